// lsg_march3.cuh — 2.5-D tiled fused stage kernel for 3-D grids (sm_100a).
//
// Block = a TX x R tile of the (x, y) plane (full rows when they fit, else
// x segments), marching along z through a balanced chunk of planes.  Each
// thread owns two x-adjacent nodes (x, x+1), so the x-window (2W+2 values) is
// shared by the pair, and every shared-memory access is a 128-bit load of a
// node pair.
//   * Planes stream through a shared-memory ring of 2W+1+D slots (D = 2
//     planes in flight) filled by cp.async: each thread copies its own pair
//     and up to kMaxHalo halo slots of a W-wide cross-shaped ring.  Halo
//     slots hold the padded-line value (in-range node, periodic wrap, or the
//     extrapolated ghost a + k*(a - b) written by a ghost pass,
//     grid.cpp:108-128), so every window is a plain read.  Ghost planes
//     beyond a global z edge are extrapolated at load time; slab halo planes
//     are read from the buffer.  One barrier per plane.
//   * The z-window of a pair is the pair's slot in the 2W+1 resident planes.
//   * L/R per dimension, central costate, H, global-LF dissipation, clamp and
//     the TVD-RK combination use exactly the arithmetic of stage_kernel, so
//     results are bit-identical to it and to the reference.
//   * The stage's v range (step log) is reduced per block (block_range).
//   * Programmatic dependent launch: set-up runs before griddepcontrol.wait.
#pragma once

#include "lsg_kernels.cuh"

namespace lsg {

struct March3 {
    int TX;      // tile width along x (even)
    int R;       // tile height along y
    int ntx;     // tiles along x
    int nzc;     // z-chunks per launch: a balanced split, the first (planes % nzc) one plane longer
    int pitch;   // shared-memory row pitch in doubles (even)
};

constexpr int kMaxHalo = 3;  // halo slots per thread (the host picks tiles that respect it)

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

__device__ __forceinline__ void cp_async8(double* dst, const double* src) {
    const unsigned d = static_cast<unsigned>(__cvta_generic_to_shared(dst));
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(d), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
    asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory");
}

// Ring geometry shared by host and device.
template <int W>
struct RingShape {
    static constexpr int D = 2;              // planes in flight ahead of the newest plane needed
    static constexpr int NB = 2 * W + 1 + D; // u planes resident: z-W .. z+W+D
    static constexpr int NV = D + 1;         // v0 planes resident: z .. z+D
    static constexpr int SH = W & 1;         // column shift: node-pair slots 16-byte aligned
    static constexpr int XW = (2 * W + 2 + SH + 1) & ~1;  // x-window doubles loaded per pair
};

// Resident blocks per SM: 3 for the narrow First/ENO2 stencils (80 registers,
// issue-bound at 512^3: +6-7 % over 2), 2 for ENO3/WENO5 (128 registers; 1 and
// 3 were measured slower).
template <int S, int KIND, int MODE, bool RANGE>
__global__ void __launch_bounds__(256, S <= ENO2 ? 3 : 2) march3_kernel(const __grid_constant__ StageParams P,
                                                                       const __grid_constant__ March3 M) {
    constexpr int W = SchemeWidth<S>::W;
    using RS = RingShape<W>;
    constexpr int D = RS::D, NB = RS::NB, NV = RS::NV, SH = RS::SH, XW = RS::XW;
    extern __shared__ __align__(16) double sm[];
    const int n0 = P.n[0], n1 = P.n[1];
    const long long s2 = P.stride[2];
    const int TX = M.TX, pitch = M.pitch, TX2 = M.TX >> 1;
    const int plane_sz = pitch * (M.R + 2 * W);
    const int vplane_sz = TX * M.R;
    double* const ring = sm;
    double* const vring = sm + NB * plane_sz;
    const int t = threadIdx.x;
    const int xt = blockIdx.x % M.ntx, yt = blockIdx.x / M.ntx;
    const int x0 = xt * TX, y0 = yt * M.R;
    const int cols = min(TX, n0 - x0), rows = min(M.R, n1 - y0);
    // logical chunk [zsl, zel) of a balanced split of [zlo, zhi): the longer
    // chunks come first in launch order, so they spread over distinct SMs in
    // the first wave.  A chunk never straddles zsplit (the host splits so),
    // so it maps to physical planes as one block.
    const int nplanes = P.zhi - P.zlo, cb = nplanes / M.nzc, crem = nplanes - cb * M.nzc;
    const int cidx = blockIdx.y;
    const int zsl = P.zlo + cidx * cb + min(cidx, crem);
    const int zel = zsl + cb + (cidx < crem ? 1 : 0);
    const int zs = zsl >= P.zsplit ? zsl + P.zskip : zsl;
    const int ze = zsl >= P.zsplit ? zel + P.zskip : min(zel, P.zsplit);
    const int yl = t / TX2, pl = t - (t / TX2) * TX2;
    const int xl = 2 * pl;
    const bool active = yl < rows && xl < cols;
    const bool two = active && xl + 1 < cols;
    const int x = x0 + (active ? xl : 0), y = y0 + (active ? yl : 0);
    const int coli = y * n0 + x;                      // in-plane offset of (x, y)
    const int me = (yl + W) * pitch + (xl + W + SH);  // own pair slot (even)
    const int vme = yl * TX + xl;                     // own pair slot in the v0 ring (even)

    // ---- halo slots: copies from global, or ghosts computed in shared memory
    const int nyh = 2 * W * cols;
    const int nxh = 2 * W * rows;
    int hsrc[kMaxHalo], hdst[kMaxHalo], ga[kMaxHalo], gb[kMaxHalo];
    double gk[kMaxHalo];
#pragma unroll
    for (int q = 0; q < kMaxHalo; ++q) {
        const int h = t + q * blockDim.x;
        hsrc[q] = -1, hdst[q] = -1, ga[q] = 0, gb[q] = 0, gk[q] = 0.0;
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
            hdst[q] = r * pitch + c + SH;
            bool ghost = false;
            if (gy < 0 || gy >= n1) {
                if (P.bc[1] == LSG_BC_PERIODIC) {
                    gy = gy < 0 ? gy + n1 : gy - n1;
                } else {  // dst[w-k] = lo + k*(lo - x1): edge rows are inside the tile
                    const int e0 = gy < 0 ? 0 : n1 - 1, e1 = gy < 0 ? 1 : n1 - 2;
                    ga[q] = (e0 - y0 + W) * pitch + c + SH;
                    gb[q] = (e1 - y0 + W) * pitch + c + SH;
                    gk[q] = (double)(gy < 0 ? -gy : gy - (n1 - 1));
                    ghost = true;
                }
            }
            if (gx < 0 || gx >= n0) {
                if (P.bc[0] == LSG_BC_PERIODIC) {
                    gx = gx < 0 ? gx + n0 : gx - n0;
                } else {
                    const int e0 = gx < 0 ? 0 : n0 - 1, e1 = gx < 0 ? 1 : n0 - 2;
                    ga[q] = r * pitch + (e0 - x0 + W) + SH;
                    gb[q] = r * pitch + (e1 - x0 + W) + SH;
                    gk[q] = (double)(gx < 0 ? -gx : gx - (n0 - 1));
                    ghost = true;
                }
            }
            if (!ghost) hsrc[q] = gy * n0 + gx;
        }
    }

    const int nglob = P.nz_glob;
    // Ring slots: u-plane p lives in slot (p - zs + W) mod NB, v0-plane p in
    // (p - zs) mod NV.  Planes are issued, ghost-filled and consumed strictly in
    // order, so each of those walks keeps its own running offset (no modulo).
    const int ring_sz = NB * plane_sz, vring_sz = NV * vplane_sz;
    int is_off = 0, vi_off = 0;  // next u / v0 plane to issue
    int gp_off = 0;              // next u plane to ghost-fill
    auto bump = [](int& off, int step, int size) {
        off += step;
        if (off == size) off = 0;
    };
    bool has_ghost = false;
#pragma unroll
    for (int q = 0; q < kMaxHalo; ++q) has_ghost |= hdst[q] >= 0 && hsrc[q] < 0;

    // Issue the async copies of u-plane p (chunk-relative window [zs-W, ze+W))
    // and of v0-plane p-W, as one commit group.
    auto issue = [&](int p) {
        if (p < ze + W) {
            double* buf = ring + is_off;
            const int zg = P.z0 + p;
            int src = p;
            bool ghost_plane = false;
            if (zg < 0 || zg >= nglob) {
                if (P.bc[2] == LSG_BC_PERIODIC) src = P.halo ? p : (zg < 0 ? p + nglob : p - nglob);
                else ghost_plane = true;
            }
            if (!ghost_plane) {
                const double* base = P.u + (long long)src * s2;
                if (active) cp_async8(buf + me, base + coli);
                if (two) cp_async8(buf + me + 1, base + coli + 1);
#pragma unroll
                for (int q = 0; q < kMaxHalo; ++q)
                    if (hsrc[q] >= 0) cp_async8(buf + hdst[q], base + hsrc[q]);
            } else {
                // extrapolated plane beyond a global boundary (grid.cpp:120-126): plain loads
                const int e0 = zg < 0 ? 0 : nglob - 1, e1 = zg < 0 ? 1 : nglob - 2;
                const double k = (double)(zg < 0 ? -zg : zg - (nglob - 1));
                const double* b0 = P.u + (long long)(e0 - P.z0) * s2;
                const double* b1 = P.u + (long long)(e1 - P.z0) * s2;
                auto ext = [&](int o) {
                    const double lo = __ldg(b0 + o);
                    return lo + k * (lo - __ldg(b1 + o));
                };
                if (active) buf[me] = ext(coli);
                if (two) buf[me + 1] = ext(coli + 1);
#pragma unroll
                for (int q = 0; q < kMaxHalo; ++q)
                    if (hsrc[q] >= 0) buf[hdst[q]] = ext(hsrc[q]);
            }
        }
        if (MODE == MODE_COMBINE) {
            const int pv = p - W;
            if (pv >= zs && pv < ze) {
                double* vb = vring + vi_off;
                bump(vi_off, vplane_sz, vring_sz);
                const double* base = P.v0 + (long long)pv * s2;
                if (active) cp_async8(vb + vme, base + coli);
                if (two) cp_async8(vb + vme + 1, base + coli + 1);
            }
        }
        cp_async_commit();
        bump(is_off, plane_sz, ring_sz);
    };
    auto ghost_pass = [&](int p) {
        if (has_ghost && p < ze + W) {
            double* buf = ring + gp_off;
#pragma unroll
            for (int q = 0; q < kMaxHalo; ++q)
                if (hdst[q] >= 0 && hsrc[q] < 0) {
                    const double a = buf[ga[q]];
                    buf[hdst[q]] = a + gk[q] * (a - buf[gb[q]]);
                }
        }
        bump(gp_off, plane_sz, ring_sz);
    };

    // Programmatic dependent launch: everything above is independent of the
    // previous stage; wait for it before the first read of its output.
    asm volatile("griddepcontrol.wait;\n" ::: "memory");

    // ---- prologue: u-planes zs-W .. zs+W+D-1 in flight, then the first 2W+1 resident
#pragma unroll 1
    for (int p = zs - W; p < zs + W + D; ++p) issue(p);
    cp_async_wait<D>();  // groups up to u-plane zs+W-1 complete
    __syncthreads();
#pragma unroll 1
    for (int p = zs - W; p < zs + W; ++p) ghost_pass(p);

    unsigned long long kmin = ~0ull, kmax = 0ull;
    unsigned fz = ~0u;  // first zero code (index << 1 | sign); padded grids < 2^31 nodes fit 32 bits
    bool bad = false;
    const double ax0 = __ldg(P.axis[0] + x), ax1 = __ldg(P.axis[0] + x + (two ? 1 : 0));
    const double ay = __ldg(P.axis[1] + y);
    double az = __ldg(P.axis[2] + P.z0 + zs);
    Trig tr = load_trig<KIND>(P, P.z0 + zs, 0);

    int j0 = 0;      // ring slot of plane z-W (advances by one per plane)
    int vr_off = 0;  // v0 ring offset of plane z
#pragma unroll 1
    for (int z = zs; z < ze; ++z) {
        cp_async_wait<D - 1>();  // u-plane z+W (and v0-plane z) complete for this thread
        __syncthreads();         // ... and for every thread; slot of z-W-1 is free
        ghost_pass(z + W);
        issue(z + W + D);
        // the 2W+1 resident planes z-W..z+W sit in ring slots j0, j0+1, ... (mod NB)
        const double* zpl[2 * W + 1];
#pragma unroll
        for (int k = 0; k < 2 * W + 1; ++k) {
            const int j = j0 + k;
            zpl[k] = ring + (j >= NB ? j - NB : j) * plane_sz + me;
        }
        j0 = j0 + 1 == NB ? 0 : j0 + 1;
        double azn = 0.0;
        Trig trn;
        if (z + 1 < ze) {
            azn = __ldg(P.axis[2] + P.z0 + z + 1);
            trn = load_trig<KIND>(P, P.z0 + z + 1, 0);
        }
        if (active) {
            const double* cur = zpl[W] - me;
            const int idx = coli + z * (int)s2;
            double L, R;
            double pa[3], pb[3];
            double da = 0.0, db = 0.0;
            {   // x: 2W+2 consecutive padded-line values shared by the pair
                double wx[XW];
                const double* xrow = cur + me - W - SH;
#pragma unroll
                for (int j = 0; j < XW; j += 2) {
                    const double2 v = *reinterpret_cast<const double2*>(xrow + j);
                    wx[j] = v.x;
                    wx[j + 1] = v.y;
                }
                double L2, R2;
                line_lr2<S>(wx + SH, P.lc[0], L, R, L2, R2);
                pa[0] = 0.5 * (L + R);
                da += P.alpha[0] * (R - L);
                pb[0] = 0.5 * (L2 + R2);
                db += P.alpha[0] * (R2 - L2);
            }
            double ca, cb;  // centre values
            {   // y: one 128-bit load per row gives both nodes' windows
                double wa[2 * W + 1], wb[2 * W + 1];
#pragma unroll
                for (int k = -W; k <= W; ++k) {
                    const double2 v = *reinterpret_cast<const double2*>(cur + me + k * pitch);
                    wa[W + k] = v.x;
                    wb[W + k] = v.y;
                }
                ca = wa[W];
                cb = wb[W];
                line_lr<S>(wa, P.lc[1], L, R);
                pa[1] = 0.5 * (L + R);
                da += P.alpha[1] * (R - L);
                line_lr<S>(wb, P.lc[1], L, R);
                pb[1] = 0.5 * (L + R);
                db += P.alpha[1] * (R - L);
            }
            {   // z: the pair's slot in the 2W+1 resident planes
                double wa[2 * W + 1], wb[2 * W + 1];
#pragma unroll
                for (int k = -W; k <= W; ++k) {
                    const double2 v = *reinterpret_cast<const double2*>(zpl[W + k]);
                    wa[W + k] = v.x;
                    wb[W + k] = v.y;
                }
                line_lr<S>(wa, P.lc[2], L, R);
                pa[2] = 0.5 * (L + R);
                da += P.alpha[2] * (R - L);
                line_lr<S>(wb, P.lc[2], L, R);
                pb[2] = 0.5 * (L + R);
                db += P.alpha[2] * (R - L);
            }
            double b0 = 0.0, b1 = 0.0;
            if (MODE == MODE_COMBINE) {
                const double2 v = *reinterpret_cast<const double2*>(vring + vr_off + vme);
                b0 = v.x;
                b1 = v.y;
            }
            double xs[3] = {ax0, ay, az};
            const double oa = finish_node<KIND, MODE>(P, xs, tr, pa, da, ca, b0, bad);
            xs[0] = ax1;
            bool bad_b = false;
            const double ob = finish_node<KIND, MODE>(P, xs, tr, pb, db, cb, b1, bad_b);
            P.out[idx] = oa;
            if (two) {
                P.out[idx + 1] = ob;
                bad |= bad_b;
            }
            if (RANGE) {
                const unsigned long long ka = order_key(oa), kb = two ? order_key(ob) : ka;
                kmin = min(kmin, min(ka, kb));
                kmax = max(kmax, max(ka, kb));
                if (oa == 0.0 || (two && ob == 0.0)) {  // rare: zeros decide the step log's sign of 0
                    const unsigned g = (unsigned)((P.z0 + z) * (int)s2 + coli);
                    const unsigned ca = (unsigned)zero_code(oa, g), cb = two ? (unsigned)zero_code(ob, g + 1) : ~0u;
                    fz = min(fz, min(ca, cb));
                }
            }
        }
        az = azn;
        tr = trn;
        bump(vr_off, vplane_sz, vring_sz);
    }
    cp_async_wait<0>();
    asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");

    if (P.flags && __any_sync(0xffffffffu, bad) && (t & 31) == 0) atomicOr(P.flags, FLAG_HAM_NONFINITE);
    if (RANGE && P.range) block_range(P.range, kmin, kmax, fz == ~0u ? ~0ull : (unsigned long long)fz);
}

using March3Fn = void (*)(StageParams, March3);

}  // namespace lsg
