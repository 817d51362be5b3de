// lsg_march3.cuh — 2.5-D tiled fused stage kernel for 3-D grids (sm_100a).
//
// Block = R full x-rows (R*n0 threads, one node each) of one y-tile, marching
// along z through a chunk of planes.  Per plane:
//   * the block stages the plane tile with W ghost rows above/below in shared
//     memory (centre rows come from the threads' registers, halo rows are
//     prefetched one plane ahead);
//   * x- and y-windows are read from shared memory with the reference's
//     ghost rules (grid.cpp:108-128) applied at the domain edges;
//   * the z-window lives in registers and slides: one new value per plane,
//     prefetched one plane ahead (ghost planes of a slab come from the halo
//     buffer planes, global ghosts from the periodic wrap / extrapolation);
//   * L/R per dimension, central costate, H, global-LF dissipation, clamp and
//     the TVD-RK combination are fused exactly as in stage_kernel, so the
//     result is bit-identical to it (and to the reference).
// No index division per node, one global load per node per plane plus the
// halo rows, one store.
#pragma once

#include "lsg_kernels.cuh"

namespace lsg {

struct March3 {
    int TX;      // tile width along x (== n0: full rows, no x-halo)
    int R;       // tile height along y
    int ntx;     // tiles along x
    int zchunk;  // planes per block
};

template <int W>
__device__ __forceinline__ double zvalue(const StageParams& P, long long base, int zz) {
    const long long s2 = P.stride[2];
    const int zg = P.z0 + zz;
    const int ng = P.nz_glob;
    if (zg >= 0 && zg < ng) return __ldg(P.u + base + zz * s2);
    if (P.bc[2] == LSG_BC_PERIODIC) {
        if (P.halo) return __ldg(P.u + base + zz * s2);
        const int zw = zg < 0 ? zg + ng : zg - ng;
        return __ldg(P.u + base + (long long)(zw - P.z0) * s2);
    }
    if (zg < 0) {
        const double lo = __ldg(P.u + base + (long long)(0 - P.z0) * s2);
        const double x1 = __ldg(P.u + base + (long long)(1 - P.z0) * s2);
        return lo + (double)(-zg) * (lo - x1);
    }
    const double hi = __ldg(P.u + base + (long long)(ng - 1 - P.z0) * s2);
    const double x2 = __ldg(P.u + base + (long long)(ng - 2 - P.z0) * s2);
    return hi + (double)(zg - (ng - 1)) * (hi - x2);
}

// Window along a line of the staged tile: node j of the global line (n
// nodes, tile origin o) sits at sm[off + (j - o + W) * st].  Out-of-range
// nodes follow the ghost rule: periodic halo slots were loaded wrapped (or,
// when the tile spans the whole line, the wrapped node is read directly);
// extrapolation uses the edge nodes, which are inside the tile whenever a
// ghost is needed (grid.cpp:108-128).
template <int W>
__device__ __forceinline__ void tile_window(const double* sm, int off, int st, int i, int o, int n, int bc,
                                            bool full, double* s) {
#pragma unroll
    for (int k = -W; k <= W; ++k) {
        const int j = i + k;
        double v;
        if (j >= 0 && j < n) {
            v = sm[off + (j - o + W) * st];
        } else if (bc == LSG_BC_PERIODIC) {
            const int jj = full ? (j < 0 ? j + n : j - n) : j;
            v = sm[off + (jj - o + W) * st];
        } else if (j < 0) {
            const double lo = sm[off + (0 - o + W) * st];
            const double x1 = sm[off + (1 - o + W) * st];
            v = lo + (double)(-j) * (lo - x1);
        } else {
            const double hi = sm[off + (n - 1 - o + W) * st];
            const double x2 = sm[off + (n - 2 - o + W) * st];
            v = hi + (double)(j - (n - 1)) * (hi - x2);
        }
        s[W + k] = v;
    }
}

constexpr int kMaxHalo = 4;  // halo slots per thread (the host picks tiles that respect it)

template <int S, int KIND, int MODE>
__global__ void __launch_bounds__(512, 1) march3_kernel(const __grid_constant__ StageParams P,
                                                         const __grid_constant__ March3 M) {
    constexpr int W = SchemeWidth<S>::W;
    extern __shared__ double sm[];
    const int n0 = P.n[0], n1 = P.n[1];
    const long long s2 = P.stride[2];
    const int TX = M.TX, pitch = M.TX + 2 * W;
    const int t = threadIdx.x;
    const int xt = blockIdx.x % M.ntx, yt = blockIdx.x / M.ntx;
    const int x0 = xt * TX, y0 = yt * M.R;
    const int cols = min(TX, n0 - x0), rows = min(M.R, n1 - y0);
    const bool fullx = TX >= n0, fully = M.R >= n1;
    const int zs = blockIdx.y * M.zchunk;
    const int ze = min(zs + M.zchunk, P.n[2]);
    const int yl = t / TX, xl = t - (t / TX) * TX;
    const bool active = yl < rows && xl < cols;
    const int x = x0 + (active ? xl : 0), y = y0 + (active ? yl : 0);
    const long long col = (long long)y * n0 + x;  // offset of (x, y, 0)
    const int me = (yl + W) * pitch + (xl + W);   // own slot

    // halo slots of the cross-shaped tile: y-halo rows, then x-halo columns
    const int nyh = 2 * W * cols;
    const int nxh = fullx ? 0 : 2 * W * rows;
    int hsrc[kMaxHalo], hdst[kMaxHalo];
#pragma unroll
    for (int q = 0; q < kMaxHalo; ++q) {
        const int h = t + q * blockDim.x;
        hsrc[q] = -1;
        hdst[q] = -1;
        int r = 0, c = 0;
        bool use = false;
        if (h < nyh) {
            const int hr = h / cols, hc = h - (h / cols) * cols;
            r = hr < W ? hr : rows + hr;
            c = W + hc;
            use = true;
        } else if (h < nyh + nxh) {
            const int g = h - nyh;
            const int hc = g / rows, hr = g - (g / rows) * rows;
            c = hc < W ? hc : cols + hc;
            r = W + hr;
            use = true;
        }
        if (use) {
            int gy = y0 - W + r, gx = x0 - W + c;
            bool ok = true;
            if (gy < 0 || gy >= n1) {
                if (P.bc[1] == LSG_BC_PERIODIC && !fully) gy = gy < 0 ? gy + n1 : gy - n1;
                else ok = false;
            }
            if (gx < 0 || gx >= n0) {
                if (P.bc[0] == LSG_BC_PERIODIC && !fullx) gx = gx < 0 ? gx + n0 : gx - n0;
                else ok = false;
            }
            if (ok) {
                hsrc[q] = gy * n0 + gx;
                hdst[q] = r * pitch + c;
            }
        }
    }

    // prologue: z-window for the first plane and its halo
    double s[2 * W + 1];
#pragma unroll
    for (int j = 0; j < 2 * W + 1; ++j) s[j] = active ? zvalue<W>(P, col, zs - W + j) : 0.0;
    double hv[kMaxHalo];
#pragma unroll
    for (int q = 0; q < kMaxHalo; ++q) hv[q] = hsrc[q] >= 0 ? __ldg(P.u + hsrc[q] + (long long)zs * s2) : 0.0;

    unsigned long long kmin = ~0ull, kmax = 0ull;
    bool bad = false;
    const double ax = __ldg(P.axis[0] + x), ay = __ldg(P.axis[1] + y);

    for (int z = zs; z < ze; ++z) {
        __syncthreads();
        if (active) sm[me] = s[W];
#pragma unroll
        for (int q = 0; q < kMaxHalo; ++q)
            if (hdst[q] >= 0) sm[hdst[q]] = hv[q];
        // prefetch the next plane's window value and halo
        double nxt = 0.0;
        if (z + 1 < ze) {
            if (active) nxt = zvalue<W>(P, col, z + 1 + W);
#pragma unroll
            for (int q = 0; q < kMaxHalo; ++q)
                if (hsrc[q] >= 0) hv[q] = __ldg(P.u + hsrc[q] + (long long)(z + 1) * s2);
        }
        __syncthreads();
        if (active) {
            const long long idx = col + (long long)z * s2;
            const int zg = P.z0 + z;
            double xs[kMaxDim] = {ax, ay, __ldg(P.axis[2] + zg), 0, 0, 0};
            int ix[kMaxDim] = {x, y, zg, 0, 0, 0};
            double p[3];
            double diss = 0.0;
            double w[2 * W + 1];
            double L, R;
            tile_window<W>(sm, (yl + W) * pitch, 1, x, x0, n0, P.bc[0], fullx, w);
            line_lr<S>(w, P.lc[0], L, R);
            p[0] = 0.5 * (L + R);
            diss += P.alpha[0] * (R - L);
            tile_window<W>(sm, xl + W, pitch, y, y0, n1, P.bc[1], fully, w);
            line_lr<S>(w, P.lc[1], L, R);
            p[1] = 0.5 * (L + R);
            diss += P.alpha[1] * (R - L);
            line_lr<S>(s, P.lc[2], L, R);
            p[2] = 0.5 * (L + R);
            diss += P.alpha[2] * (R - L);
            const double H = hamiltonian<KIND, 3>(P, xs, ix, p);
            bad |= !isfinite(H);
            double dv = -(H - 0.5 * diss);
            if (P.restrict_update) dv = P.direction == LSG_GROW ? ((0.0 < dv) ? 0.0 : dv) : ((dv < 0.0) ? 0.0 : dv);
            double o;
            if constexpr (MODE == MODE_TERM) {
                o = dv;
            } else if constexpr (MODE == MODE_EULER) {
                o = s[W] + P.dt * dv;
            } else {
                const double base = P.v0[idx];
                o = base + P.c * ((s[W] + P.dt * dv) - base);
            }
            P.out[idx] = o;
            const unsigned long long key = order_key(o);
            kmin = min(kmin, key);
            kmax = max(kmax, key);
        }
#pragma unroll
        for (int j = 0; j < 2 * W; ++j) s[j] = s[j + 1];
        s[2 * W] = nxt;
    }

    if (P.flags && __any_sync(0xffffffffu, bad) && (t & 31) == 0) atomicOr(P.flags, FLAG_HAM_NONFINITE);
    if (P.range) {
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) {
            kmin = min(kmin, __shfl_xor_sync(0xffffffffu, kmin, off));
            kmax = max(kmax, __shfl_xor_sync(0xffffffffu, kmax, off));
        }
        __shared__ unsigned long long rmin[32], rmax[32];
        const int warp = t >> 5, lane = t & 31;
        if (lane == 0) {
            rmin[warp] = kmin;
            rmax[warp] = kmax;
        }
        __syncthreads();
        if (warp == 0) {
            const int nw = blockDim.x >> 5;
            kmin = lane < nw ? rmin[lane] : ~0ull;
            kmax = lane < nw ? rmax[lane] : 0ull;
#pragma unroll
            for (int off = 16; off > 0; off >>= 1) {
                kmin = min(kmin, __shfl_xor_sync(0xffffffffu, kmin, off));
                kmax = max(kmax, __shfl_xor_sync(0xffffffffu, kmax, off));
            }
            if (lane == 0) {
                if (kmin != ~0ull) atomicMax(P.range, ~kmin);
                if (kmax != 0ull) atomicMax(P.range + 1, kmax);
            }
        }
    }
}

using March3Fn = void (*)(StageParams, March3);

}  // namespace lsg
