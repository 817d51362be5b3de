// lsg_march3.cuh — 2.5-D tiled fused stage kernel for 3-D grids (sm_100a).
//
// Block = a TX x R tile of the (x, y) plane, marching along z through a chunk
// of planes.  Each thread owns two x-adjacent nodes (x, x+1), so the x-window
// (2W+2 values) is shared by the pair, and every shared-memory access is a
// 128-bit load of a node pair.  Per plane:
//   * the tile and a W-wide halo ring (cross-shaped, no corners) are staged in
//     shared memory: centre pairs come from the threads' registers, halo slots
//     are prefetched one plane ahead and already hold the padded-line value
//     (in-range node, periodic wrap, or the extrapolated ghost
//     a + k*(a - b), grid.cpp:108-128), so every window is a plain read;
//   * the z-windows of both nodes live in registers and slide one plane,
//     the next value prefetched one plane ahead (slab halo planes / global
//     ghosts resolved at load time, uniformly per block);
//   * L/R per dimension, central costate, H, global-LF dissipation, clamp and
//     the TVD-RK combination use exactly the arithmetic of stage_kernel, so
//     results are bit-identical to it and to the reference.
#pragma once

#include "lsg_kernels.cuh"

namespace lsg {

struct March3 {
    int TX;      // tile width along x (even)
    int R;       // tile height along y
    int ntx;     // tiles along x
    int zchunk;  // planes per block
    int pitch;   // shared-memory row pitch in doubles (even)
};

constexpr int kMaxHalo = 4;  // halo slots per thread (the host picks tiles that respect it)

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

// Finish one node: H, dissipation, clamp, RK combination; returns the output.
template <int KIND, int MODE>
__device__ __forceinline__ double finish_node(const StageParams& P, const double* xs, const Trig& tr,
                                              const double* p, double diss, double centre, double base,
                                              bool& bad) {
    const double H = hamiltonian<KIND, 3>(P, xs, tr, p);
    bad |= !isfinite(H);
    double dv = -(H - 0.5 * diss);
    if (P.restrict_update) dv = P.direction == LSG_GROW ? ((0.0 < dv) ? 0.0 : dv) : ((dv < 0.0) ? 0.0 : dv);
    if constexpr (MODE == MODE_TERM) {
        return dv;
    } else if constexpr (MODE == MODE_EULER) {
        return centre + P.dt * dv;
    } else {
        return base + P.c * ((centre + P.dt * dv) - base);
    }
}

template <int S, int KIND, int MODE, bool RANGE>
__global__ void __launch_bounds__(256, 2) march3_kernel(const __grid_constant__ StageParams P,
                                                         const __grid_constant__ March3 M) {
    constexpr int W = SchemeWidth<S>::W;
    constexpr int SH = W & 1;                      // column shift that makes pair slots 16-byte aligned
    constexpr int XW = (2 * W + 2 + SH + 1) & ~1;  // x-window doubles loaded (even)
    extern __shared__ __align__(16) double sm[];
    const int n0 = P.n[0], n1 = P.n[1];
    const long long s2 = P.stride[2];
    const int s2i = (int)s2;  // the host only picks this kernel for slabs below 2^31 nodes
    const int TX = M.TX, pitch = M.pitch, TX2 = M.TX >> 1;
    const int t = threadIdx.x;
    const int xt = blockIdx.x % M.ntx, yt = blockIdx.x / M.ntx;
    const int x0 = xt * TX, y0 = yt * M.R;
    const int cols = min(TX, n0 - x0), rows = min(M.R, n1 - y0);
    const int zs = blockIdx.y * M.zchunk;
    const int ze = min(zs + M.zchunk, P.n[2]);
    const int yl = t / TX2, pl = t - (t / TX2) * TX2;
    const int xl = 2 * pl;
    const bool active = yl < rows && xl < cols;
    const bool two = active && xl + 1 < cols;
    const int x = x0 + (active ? xl : 0), y = y0 + (active ? yl : 0);
    const long long col = (long long)y * n0 + x;      // offset of (x, y, 0)
    const int coli = y * n0 + x;
    const int me = (yl + W) * pitch + (xl + W + SH);  // own pair slot (even)

    // ---- halo slots ---------------------------------------------------------
    const int nyh = 2 * W * cols;
    const int nxh = 2 * W * rows;
    int hpa[kMaxHalo], hpb[kMaxHalo];  // 32-bit in-plane node offsets (-1: none)
    int hdst[kMaxHalo];
    double hk[kMaxHalo];
#pragma unroll
    for (int q = 0; q < kMaxHalo; ++q) {
        const int h = t + q * blockDim.x;
        hpa[q] = -1;
        hpb[q] = -1;
        hdst[q] = -1;
        hk[q] = 0.0;
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
            const int gy = y0 - W + r, gx = x0 - W + c;
            int sy = gy, sx = gx, ey = -1, ex = -1;
            if (gy < 0 || gy >= n1) {
                if (P.bc[1] == LSG_BC_PERIODIC) {
                    sy = gy < 0 ? gy + n1 : gy - n1;
                } else if (gy < 0) {
                    sy = 0, ey = 1, hk[q] = (double)(-gy);
                } else {
                    sy = n1 - 1, ey = n1 - 2, hk[q] = (double)(gy - (n1 - 1));
                }
            }
            if (gx < 0 || gx >= n0) {
                if (P.bc[0] == LSG_BC_PERIODIC) {
                    sx = gx < 0 ? gx + n0 : gx - n0;
                } else if (gx < 0) {
                    sx = 0, ex = 1, hk[q] = (double)(-gx);
                } else {
                    sx = n0 - 1, ex = n0 - 2, hk[q] = (double)(gx - (n0 - 1));
                }
            }
            hpa[q] = sy * n0 + sx;
            if (ey >= 0) hpb[q] = ey * n0 + sx;
            if (ex >= 0) hpb[q] = sy * n0 + ex;
            hdst[q] = r * pitch + c + SH;
        }
    }

    // ---- prologue ------------------------------------------------------------
    double s0[2 * W + 1], s1[2 * W + 1];
#pragma unroll
    for (int j = 0; j < 2 * W + 1; ++j) {
        s0[j] = active ? zvalue<W>(P, col, zs - W + j) : 0.0;
        s1[j] = two ? zvalue<W>(P, col + 1, zs - W + j) : 0.0;
    }
    // Raw halo values (the ghost formula is applied when staging, so loads stay
    // in flight): ha/hb hold the plane staged next.
    double ha[kMaxHalo], hb[kMaxHalo];
    auto load_halo = [&](int zz) {
        const int off = zz * s2i;
#pragma unroll
        for (int q = 0; q < kMaxHalo; ++q) {
            if (hpa[q] >= 0) ha[q] = __ldg(P.u + (hpa[q] + off));
            if (hpb[q] >= 0) hb[q] = __ldg(P.u + (hpb[q] + off));
        }
    };
    auto stage_plane = [&](double* buf, double c0, double c1) {
        if (two) *reinterpret_cast<double2*>(buf + me) = make_double2(c0, c1);
        else if (active) buf[me] = c0;  // me+1 is a ghost slot the halo pass fills
#pragma unroll
        for (int q = 0; q < kMaxHalo; ++q)
            if (hdst[q] >= 0) buf[hdst[q]] = hpb[q] >= 0 ? ha[q] + hk[q] * (ha[q] - hb[q]) : ha[q];
    };
#pragma unroll
    for (int q = 0; q < kMaxHalo; ++q) ha[q] = hb[q] = 0.0;
    load_halo(zs);
    double* const bufs[2] = {sm, sm + pitch * (M.R + 2 * W)};
    stage_plane(bufs[0], s0[W], s1[W]);
    if (zs + 1 < ze) load_halo(zs + 1);

    unsigned long long kmin = ~0ull, kmax = 0ull;
    bool bad = false;
    const double ax0 = __ldg(P.axis[0] + x), ax1 = __ldg(P.axis[0] + x + (two ? 1 : 0));
    const double ay = __ldg(P.axis[1] + y);
    // planes z whose prefetch target z+1+W is a real in-slab plane need no ghost logic
    const int zfast_lo = -P.z0 - 1 - W;
    const int zfast_hi = P.nz_glob - P.z0 - 2 - W;
    // per-plane operands, prefetched one plane ahead
    double az = __ldg(P.axis[2] + P.z0 + zs);
    Trig tr = load_trig<KIND>(P, P.z0 + zs, 0);
    double b0 = 0.0, b1 = 0.0;
    if (MODE == MODE_COMBINE && active) {
        const int o = coli + zs * s2i;
        b0 = P.v0[o];
        b1 = P.v0[o + (two ? 1 : 0)];
    }
    __syncthreads();

    for (int z = zs; z < ze; ++z) {
        double* const cur = bufs[(z - zs) & 1];
        // stage plane z+1 into the other buffer (its centre is already in the window)
        if (z + 1 < ze) {
            stage_plane(bufs[(z - zs + 1) & 1], s0[W + 1], s1[W + 1]);
            if (z + 2 < ze) load_halo(z + 2);
        }
        // prefetch the next window value and the next plane's operands
        double n0v = 0.0, n1v = 0.0, azn = 0.0, nb0 = 0.0, nb1 = 0.0;
        Trig trn;
        if (z + 1 < ze) {
            const int zn = z + 1 + W;
            if (z >= zfast_lo && z <= zfast_hi) {  // uniform across the block
                const int o = coli + zn * s2i;
                if (active) {
                    n0v = __ldg(P.u + o);
                    n1v = __ldg(P.u + (o + (two ? 1 : 0)));
                }
            } else {
                if (active) n0v = zvalue<W>(P, col, zn);
                if (two) n1v = zvalue<W>(P, col + 1, zn);
            }
            azn = __ldg(P.axis[2] + P.z0 + z + 1);
            trn = load_trig<KIND>(P, P.z0 + z + 1, 0);
            if (MODE == MODE_COMBINE && active) {
                const int o = coli + (z + 1) * s2i;
                nb0 = P.v0[o];
                nb1 = P.v0[o + (two ? 1 : 0)];
            }
        }
        if (active) {
            const int idx = coli + z * s2i;
            const int me_ = me;
            double L, R;
            double pa[3], pb[3];
            double da = 0.0, db = 0.0;
            // x: 2W+2 consecutive padded-line values shared by the pair
            double wx[XW];
            const double* xrow = cur + me_ - W - SH;  // even (16-byte aligned) start
#pragma unroll
            for (int j = 0; j < XW; j += 2) {
                const double2 v = *reinterpret_cast<const double2*>(xrow + j);
                wx[j] = v.x;
                wx[j + 1] = v.y;
            }
            line_lr<S>(wx + SH, P.lc[0], L, R);
            pa[0] = 0.5 * (L + R);
            da += P.alpha[0] * (R - L);
            line_lr<S>(wx + SH + 1, P.lc[0], L, R);
            pb[0] = 0.5 * (L + R);
            db += P.alpha[0] * (R - L);
            // y: one 128-bit load per row gives both nodes' windows
            double ya[2 * W + 1], yb[2 * W + 1];
#pragma unroll
            for (int k = -W; k <= W; ++k) {
                const double2 v = *reinterpret_cast<const double2*>(cur + me_ + k * pitch);
                ya[W + k] = v.x;
                yb[W + k] = v.y;
            }
            line_lr<S>(ya, P.lc[1], L, R);
            pa[1] = 0.5 * (L + R);
            da += P.alpha[1] * (R - L);
            line_lr<S>(yb, P.lc[1], L, R);
            pb[1] = 0.5 * (L + R);
            db += P.alpha[1] * (R - L);
            // z: register windows
            line_lr<S>(s0, P.lc[2], L, R);
            pa[2] = 0.5 * (L + R);
            da += P.alpha[2] * (R - L);
            line_lr<S>(s1, P.lc[2], L, R);
            pb[2] = 0.5 * (L + R);
            db += P.alpha[2] * (R - L);
            double xs[3] = {ax0, ay, az};
            const double oa = finish_node<KIND, MODE>(P, xs, tr, pa, da, s0[W], b0, bad);
            xs[0] = ax1;
            bool bad_b = false;
            const double ob = finish_node<KIND, MODE>(P, xs, tr, pb, db, s1[W], b1, bad_b);
            P.out[idx] = oa;
            if (two) {
                P.out[idx + 1] = ob;
                bad |= bad_b;
            }
            if (RANGE) {
                const unsigned long long ka = order_key(oa), kb = two ? order_key(ob) : ka;
                kmin = min(kmin, min(ka, kb));
                kmax = max(kmax, max(ka, kb));
            }
        }
#pragma unroll
        for (int j = 0; j < 2 * W; ++j) {
            s0[j] = s0[j + 1];
            s1[j] = s1[j + 1];
        }
        s0[2 * W] = n0v;
        s1[2 * W] = n1v;
        az = azn;
        tr = trn;
        b0 = nb0;
        b1 = nb1;
        __syncthreads();  // plane z+1 staged; everyone is done reading plane z's buffer
    }

    if (P.flags && __any_sync(0xffffffffu, bad) && (t & 31) == 0) atomicOr(P.flags, FLAG_HAM_NONFINITE);
    if (RANGE && P.range) {
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
