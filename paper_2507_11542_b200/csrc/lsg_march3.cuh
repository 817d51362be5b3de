// lsg_march3.cuh — 2.5-D tiled fused stage kernels for 3-D grids (sm_100a):
// march3_tma_kernel (rows of an even number of doubles: each plane of a tile
// arrives by one cp.async.bulk.tensor.3d on an mbarrier ring; see its own
// comment below) and march3_kernel (any rows: per-thread cp.async), sharing
// the per-pair arithmetic (march3_pair).  What follows describes both.
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

#include <cuda.h>  // CUtensorMap (the type only; maps are encoded on the host)

#include "lsg_kernels.cuh"

namespace lsg {

struct March3 {
    int TX;      // tile width along x (even)
    int R;       // tile height along y
    int ntx;     // tiles along x
    int nzc;     // z-chunks per launch: a balanced split, the first (planes % nzc) one plane longer
    int pitch;   // shared-memory row pitch in doubles (even)
    int slot;    // march3_tma_kernel: u-ring slot stride in doubles (a multiple of 16: 128-byte TMA destinations)
    int vslot;   // ... v0-ring slot stride
    int hmax;    // ... halo cells per tile (staging slot size)
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

// ENO3 divided differences along z carried in registers from one plane to
// the next (march3_tma_kernel): at plane z the window is s[0..6] = planes
// z-3..z+3 and the selection needs d1[2..3], d2[2..4], d3[1..4]
// (spatial_derivatives.cpp:136-197); moving to z+1 every table shifts by one
// entry, so only d1[5], d2[5], d3[4] and the newest plane value are new.
// Same expressions on the same operands as the full recomputation, so the
// same bits; 6 FP64 instructions per node instead of 30.
struct Eno3Z {
    double s6;            // newest plane value s[6]
    double d1[3];         // d1[3..5]
    double d2[3];         // d2[3..5]
    double d3[3];         // d3[2..4]
};

__device__ __forceinline__ void eno3_z_init(const double* s, const LineConst& c, Eno3Z& q) {
    double d1[6], d2[6], d3[5];
#pragma unroll
    for (int j = 0; j < 6; ++j) d1[j] = (s[j + 1] - s[j]) * c.inv_dx;
#pragma unroll
    for (int j = 1; j < 6; ++j) d2[j] = (d1[j] - d1[j - 1]) * c.half_inv;
#pragma unroll
    for (int j = 1; j < 5; ++j) d3[j] = (d2[j + 1] - d2[j]) * c.third_inv;
    q.s6 = s[6];
    q.d1[0] = d1[3], q.d1[1] = d1[4], q.d1[2] = d1[5];
    q.d2[0] = d2[3], q.d2[1] = d2[4], q.d2[2] = d2[5];
    q.d3[0] = d3[2], q.d3[1] = d3[3], q.d3[2] = d3[4];
}

// L/R at plane z from the carry of plane z-1 and the new plane value s6 = s[z+3].
__device__ __forceinline__ void eno3_z_step(double s6, const LineConst& c, Eno3Z& q, double& L, double& R) {
    double d1[6], d2[6], d3[5];
    // plane z's d1[2..4] = plane z-1's d1[3..5], and so on
    d1[2] = q.d1[0], d1[3] = q.d1[1], d1[4] = q.d1[2];
    d1[5] = (s6 - q.s6) * c.inv_dx;
    d2[2] = q.d2[0], d2[3] = q.d2[1], d2[4] = q.d2[2];
    d2[5] = (d1[5] - d1[4]) * c.half_inv;
    d3[1] = q.d3[0], d3[2] = q.d3[1], d3[3] = q.d3[2];
    d3[4] = (d2[5] - d2[4]) * c.third_inv;
    q.s6 = s6;
    q.d1[0] = d1[3], q.d1[1] = d1[4], q.d1[2] = d1[5];
    q.d2[0] = d2[3], q.d2[1] = d2[4], q.d2[2] = d2[5];
    q.d3[0] = d3[2], q.d3[1] = d3[3], q.d3[2] = d3[4];
    eno3_select(d1, d2, d3, c, L, R);
}

// One node pair (x, x+1) of plane z: L/R per dimension from the shared-memory
// windows (x: the pair's row, y: its column of rows, z: its slot in the 2W+1
// resident planes zpl[]), central costate, H, dissipation, clamp, RK
// combination, the output store and the step's range candidates.
// ZC (ENO3 only): z tables carried in qa/qb (first: the chunk's first plane,
// which fills them from the full window).
// YP: the y-direction costates and dissipation terms of the pair come
// precomputed (ypr[0], ypr[1]: (p, alpha*(R-L)) per node, the y pass of march3_tma_kernel).
// ZP: z lines two planes at a time: on zeven planes both nodes' z lines
// cover planes z and z+1 (line_lr2 over zpl[0..2W+1]) and plane z+1's terms
// go to zst[0..1]; on the other planes they come from there.
template <int S, int KIND, int MODE, bool RANGE, bool ZC = false, bool YP = false, bool ZP = false>
__device__ __forceinline__ void march3_pair(const StageParams& P, const double* const* zpl, int me, int pitch,
                                            const double* vpair, int coli, int z, bool two, double ax0, double ax1,
                                            double ay, double az, const Trig& tr, unsigned long long& kmin,
                                            unsigned long long& kmax, unsigned& fz, bool& bad, Eno3Z* qa = nullptr,
                                            Eno3Z* qb = nullptr, bool first = true, const double2* ypr = nullptr,
                                            double2* zst = nullptr, bool zeven = true) {
    constexpr int W = SchemeWidth<S>::W;
    using RS = RingShape<W>;
    constexpr int SH = RS::SH, XW = RS::XW;
    const long long s2 = P.stride[2];
    const double* cur = zpl[W] - me;
    const int idx = coli + z * (int)s2;
    LSG_CHECK(idx >= 0 && idx + (two ? 1 : 0) < P.n_local);
    LSG_CHECK(me - W * pitch - W - SH >= 0);
    double L, R;
    double pa[3], pb[3];
    double da = 0.0, db = 0.0;
    double ca, cb;  // centre values
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
        costate<S>(P, 0, L, R, pa[0], da);
        costate<S>(P, 0, L2, R2, pb[0], db);
        ca = wx[W + SH];
        cb = wx[W + SH + 1];
    }
    if constexpr (YP) {
        const double2 ya = ypr[0], yb = ypr[1];
        pa[1] = ya.x;
        da += ya.y;
        pb[1] = yb.x;
        db += yb.y;
    } else {   // y: one 128-bit load per row gives both nodes' windows
        double wa[2 * W + 1], wb[2 * W + 1];
#pragma unroll
        for (int k = -W; k <= W; ++k) {
            const double2 v = *reinterpret_cast<const double2*>(cur + me + k * pitch);
            wa[W + k] = v.x;
            wb[W + k] = v.y;
        }
        line_lr<S>(wa, P.lc[1], L, R);
        costate<S>(P, 1, L, R, pa[1], da);
        line_lr<S>(wb, P.lc[1], L, R);
        costate<S>(P, 1, L, R, pb[1], db);
    }
    if (ZC && S == ENO3 && !first) {  // z: carried tables + the newest plane
        const double2 v = *reinterpret_cast<const double2*>(zpl[2 * W]);
        eno3_z_step(v.x, P.lc[2], *qa, L, R);
        costate<S>(P, 2, L, R, pa[2], da);
        eno3_z_step(v.y, P.lc[2], *qb, L, R);
        costate<S>(P, 2, L, R, pb[2], db);
    } else if (ZP && zeven) {  // z: planes z and z+1 of both nodes
        double wa[2 * W + 2], wb[2 * W + 2];
#pragma unroll
        for (int k = 0; k < 2 * W + 2; ++k) {
            const double2 v = *reinterpret_cast<const double2*>(zpl[k]);
            wa[k] = v.x;
            wb[k] = v.y;
        }
        double L1, R1, p1, t1;
        line_lr2<S>(wa, P.lc[2], L, R, L1, R1);
        costate<S>(P, 2, L, R, pa[2], da);
        costate_term<S>(P, 2, L1, R1, p1, t1);
        zst[0] = make_double2(p1, t1);
        line_lr2<S>(wb, P.lc[2], L, R, L1, R1);
        costate<S>(P, 2, L, R, pb[2], db);
        costate_term<S>(P, 2, L1, R1, p1, t1);
        zst[1] = make_double2(p1, t1);
    } else if (ZP) {
        const double2 za = zst[0], zb = zst[1];
        pa[2] = za.x;
        da += za.y;
        pb[2] = zb.x;
        db += zb.y;
    } else {   // z: the pair's slot in the 2W+1 resident planes
        double wa[2 * W + 1], wb[2 * W + 1];
#pragma unroll
        for (int k = -W; k <= W; ++k) {
            const double2 v = *reinterpret_cast<const double2*>(zpl[W + k]);
            wa[W + k] = v.x;
            wb[W + k] = v.y;
        }
        line_lr<S>(wa, P.lc[2], L, R);
        costate<S>(P, 2, L, R, pa[2], da);
        line_lr<S>(wb, P.lc[2], L, R);
        costate<S>(P, 2, L, R, pb[2], db);
        if constexpr (ZC && S == ENO3) {
            eno3_z_init(wa, P.lc[2], *qa);
            eno3_z_init(wb, P.lc[2], *qb);
        }
    }
    double b0 = 0.0, b1 = 0.0;
    if (MODE == MODE_COMBINE) {
        const double2 v = *reinterpret_cast<const double2*>(vpair);
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

// Resident blocks per SM: 3 for the narrow First/ENO2 stencils (80 registers,
// issue-bound at 512^3: +6-7 % over 2), 2 for ENO3/WENO5 (128 registers; 1 and
// 3 were measured slower).
template <int S, int KIND, int MODE, bool RANGE>
__global__ void __launch_bounds__(256, S <= ENO2 ? 3 : 2) march3_kernel(const __grid_constant__ StageParams P,
                                                                       const __grid_constant__ March3 M) {
    constexpr int W = SchemeWidth<S>::W;
    using RS = RingShape<W>;
    constexpr int D = RS::D, NB = RS::NB, NV = RS::NV, SH = RS::SH;
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
        if (active)
            march3_pair<S, KIND, MODE, RANGE>(P, zpl, me, pitch, MODE == MODE_COMBINE ? vring + vr_off + vme : nullptr,
                                              coli, z, two, ax0, ax1, ay, az, tr, kmin, kmax, fz, bad);
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

// ---- TMA-fed variant ----------------------------------------------------------
// The same tile, ring and per-pair arithmetic as march3_kernel, but each plane
// of the tile (TX + 2W + 2*SH columns, so node pairs stay 16-byte aligned,
// x R + 2W rows) arrives in one cp.async.bulk.tensor.3d issued by one thread
// and completing on the slot's mbarrier, together with the v0 plane
// (COMBINE).  The tensor map covers the slab buffer including its halo
// planes; coordinates outside the grid fill with zeros, and only tiles on
// the x/y border fix those cells up: periodic wraps through cp.async into a
// staging row (copied in after the wait), extrapolated ghosts
// (grid.cpp:108-128) computed in shared memory.  Planes beyond a global z
// edge are extrapolated by the threads as in march3_kernel.  Needs rows of an
// even number of doubles (16-byte global strides); other grids use
// march3_kernel.
// Planes in flight of the TMA ring (the host sizes shared memory to match).
// The exact WENO5 spends ~5 us per plane, so one plane in flight hides the
// load (25.03 -> 25.09 G at 512^3) and frees 11 KB of shared memory.
template <int S>
struct TmaDepth {
    static constexpr int D = S == WENO5 ? 1 : 2;
};

__device__ __forceinline__ unsigned smem_u32(const void* p) {
    return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(unsigned long long* bar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(unsigned long long* bar, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, unsigned parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra WAIT_%=;\n}\n" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* map, unsigned long long* bar, int c0, int c1,
                                            int c2) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5}], [%2];\n" ::
            "r"(smem_u32(dst)),
        "l"(reinterpret_cast<unsigned long long>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2)
        : "memory");
}

__device__ __forceinline__ void mbar_arrive(unsigned long long* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(bar)) : "memory");
}

template <int S, int KIND, int MODE, bool RANGE>
__global__ void __launch_bounds__(256, S <= ENO2 ? 3 : 2)
    march3_tma_kernel(const __grid_constant__ StageParams P, const __grid_constant__ March3 M,
                      const __grid_constant__ CUtensorMap tmu, const __grid_constant__ CUtensorMap tmv) {
    constexpr int W = SchemeWidth<S>::W;
    using RS = RingShape<W>;
    constexpr int D = TmaDepth<S>::D, NB = 2 * W + 1 + D, NV = D + 1, SH = RS::SH;
    constexpr int XL = W + SH;  // box columns start XL left of the tile
    constexpr int NS = D + 1;   // staging slots (planes whose wrap cells are in flight)
    // y pass (WENO5, both forms): the y-direction L/R of each plane computed
    // once per column pair of rows (two y-adjacent nodes share their window
    // and, in line_lr2, their differences and quotients) by thread
    // (t % TX, t / TX), one plane ahead of the pairs that use them.  Measured
    // at 512^3: exact WENO5 23.11 -> 23.78 G, fast 57.9 -> 58.5 G; ENO3 (issue-
    // bound, its y line is cheap) 83.4 -> 83.2 G, so ENO3 keeps the pair's own y.
    constexpr bool YP = S >= WENO5;
    // z pairs (fast WENO5): each pair's z lines two planes at a time
    // (march3_pair ZP), waiting for plane z+W+1 on even planes of the chunk;
    // the second plane's terms wait in a per-thread shared-memory slot.
    // 512^3: fast 58.6 -> 59.6 G; the exact WENO5 spills with it (23.8 ->
    // 22.7 G), so it keeps one z line per node and plane.  (A separate z pass
    // before the pair's work, both planes' terms through shared memory, lost:
    // fast 51.2 G, exact 22.4 G.)
    constexpr bool ZP = S == WENO5F;
    static_assert(NV == D + 1 && NB == 2 * W + D + 1 && NB <= 32, "ring geometry");
    extern __shared__ __align__(16) double sm[];
    const int n0 = P.n[0], n1 = P.n[1];
    const long long s2 = P.stride[2];
    const int TX = M.TX, pitch = M.pitch, TX2 = M.TX >> 1, slot = M.slot;
    // TMA destinations are 128-byte aligned (the host adds 128 bytes of slack);
    // offset arithmetic on the shared array keeps the accesses LDS
    double* const ring = sm + (((128u - (smem_u32(sm) & 127u)) & 127u) >> 3);
    double* const vring = ring + NB * slot;
    double* const stage = vring + NV * M.vslot;
    // YP: two (p, alpha*(R-L)) buffers of the y direction, one per plane parity
    double2* const ybuf = reinterpret_cast<double2*>(stage + NS * M.hmax);
    double2* const zst = ybuf + (YP ? 2 * TX * M.R : 0) + 2 * threadIdx.x;
    unsigned long long* const bar = reinterpret_cast<unsigned long long*>(
        stage + NS * M.hmax + (YP ? 4 * TX * M.R : 0) + (ZP ? 4 * (int)blockDim.x : 0));
    const int t = threadIdx.x;
    const int xt = blockIdx.x % M.ntx, yt = blockIdx.x / M.ntx;
    const int x0 = xt * TX, y0 = yt * M.R;
    const int cols = min(TX, n0 - x0), rows = min(M.R, n1 - y0);
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
    const int coli = y * n0 + x;
    const int me = (yl + W) * pitch + (xl + XL);  // own pair slot (even)
    const int vme = yl * TX + xl;
    const int nglob = P.nz_glob;
    // tiles whose cross-shaped halo leaves the grid, and chunks whose window
    // crosses a non-periodic global z edge, write parts of the ring from the
    // threads (block-uniform); all other tiles take every plane from TMA alone
    const bool border = x0 - W < 0 || x0 + cols + W > n0 || y0 - W < 0 || y0 + rows + W > n1;
    const bool generic_writes =
        border || (P.bc[2] != LSG_BC_PERIODIC && (P.z0 + zs - W < 0 || P.z0 + ze + W + D > nglob));
    const int nyh = 2 * W * cols, nh = nyh + 2 * W * rows;
    // y-pass item: column yc, rows yr and yr+1 (the host picks even R with
    // TX * R / 2 <= blockDim.x)
    const int yc = t % TX, yr = 2 * (t / TX);
    const bool yact = YP && yr < rows && yc < cols, ytwo = yact && yr + 1 < rows;
    const int yoff = yr * pitch + yc + XL;  // slot row yr = tile row yr - W: the window's first value
    const int yo = yr * TX + yc;
    auto ypass = [&](const double* buf, double2* dst) {
        if constexpr (YP) {
            if (!yact) return;
            double w[2 * W + 2];
#pragma unroll
            for (int k = 0; k < 2 * W + 2; ++k) w[k] = buf[yoff + k * pitch];
            double La, Ra, Lb, Rb, p, term;
            line_lr2<S>(w, P.lc[1], La, Ra, Lb, Rb);
            costate_term<S>(P, 1, La, Ra, p, term);
            dst[yo] = make_double2(p, term);
            if (ytwo) {
                costate_term<S>(P, 1, Lb, Rb, p, term);
                dst[yo + TX] = make_double2(p, term);
            }
        }
    };

#ifdef LSG_CHECKED
    {
        unsigned dyn = 0;
        asm("mov.u32 %0, %%dynamic_smem_size;" : "=r"(dyn));
        LSG_CHECK(!YP || (M.R % 2 == 0 && TX * M.R <= 2 * (int)blockDim.x));
        LSG_CHECK(!yact || yoff + (2 * W + 1) * pitch < slot);
        LSG_CHECK((smem_u32(ring) & 127u) == 0u);
        LSG_CHECK(reinterpret_cast<const char*>(bar + NB) <= reinterpret_cast<const char*>(sm) + dyn);
        LSG_CHECK(!active || (me + 1 + W * pitch < slot && vme + 1 < M.vslot));  // padding threads never read
        LSG_CHECK((me - W - SH) % 2 == 0);
    }
#endif
    if (t == 0) {
        for (int j = 0; j < NB; ++j) mbar_init(bar + j, 1);
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    __syncthreads();

    // halo cell h of the cross-shaped ring (y-halo rows first, then x-halo
    // columns): its offset in a slot and global (x, y); true when out of range
    auto halo_cell = [&](int h, int& off, int& gx, int& gy) {
        int r, c;
        if (h < nyh) {
            const int hr = h / cols, hc = h - hr * cols;
            r = hr < W ? hr : rows + hr;
            c = W + hc;
        } else {
            const int g = h - nyh;
            const int hc = g / rows, hr = g - hc * rows;
            c = hc < W ? hc : cols + hc;
            r = W + hr;
        }
        off = r * pitch + c + SH;
        gx = x0 - W + c;
        gy = y0 - W + r;
        return gx < 0 || gx >= n0 || gy < 0 || gy >= n1;
    };

    // This thread's out-of-range halo cells of a border tile (at most kMaxHalo):
    // slot offset, and either the wrapped in-plane source (periodic) or the two
    // in-tile operands and the distance of the extrapolated ghost
    // (grid.cpp:108-128), packed as b = eb | k << 24.
    int c_off[kMaxHalo], c_a[kMaxHalo], c_b[kMaxHalo];
#pragma unroll
    for (int q = 0; q < kMaxHalo; ++q) {
        c_off[q] = -1, c_a[q] = 0, c_b[q] = -1;
        const int h = t + q * blockDim.x;
        int off, gx, gy;
        if (!border || h >= nh || !halo_cell(h, off, gx, gy)) continue;
        c_off[q] = off;
        const bool wx = gx < 0 || gx >= n0;
        LSG_CHECK(off >= 0 && off < slot && h < M.hmax);
        if (wx ? P.bc[0] == LSG_BC_PERIODIC : P.bc[1] == LSG_BC_PERIODIC) {
            gx = gx < 0 ? gx + n0 : (gx >= n0 ? gx - n0 : gx);
            gy = gy < 0 ? gy + n1 : (gy >= n1 ? gy - n1 : gy);
            c_a[q] = gy * n0 + gx;
            LSG_CHECK(c_a[q] >= 0 && c_a[q] < n0 * n1);
        } else if (wx) {
            c_a[q] = off + ((gx < 0 ? 0 : n0 - 1) - gx);
            c_b[q] = (off + ((gx < 0 ? 1 : n0 - 2) - gx)) | ((gx < 0 ? -gx : gx - (n0 - 1)) << 24);
        } else {
            c_a[q] = off + ((gy < 0 ? 0 : n1 - 1) - gy) * pitch;
            c_b[q] = (off + ((gy < 0 ? 1 : n1 - 2) - gy) * pitch) | ((gy < 0 ? -gy : gy - (n1 - 1)) << 24);
        }
    }

    // Issue plane p (u-plane p into u slot j, v0-plane p-W into v0 slot vj).
    auto issue = [&](int p, int j, int vj, int sj) {
        const int zg = P.z0 + p;
        const bool outside = zg < 0 || zg >= nglob;
        const bool ghost_plane = outside && P.bc[2] != LSG_BC_PERIODIC;
        const bool want_u = p < ze + W;
        const int src = outside && !ghost_plane ? (P.halo ? p : (zg < 0 ? p + nglob : p - nglob)) : p;
        if (t == 0) {
            const int pv = p - W;
            const bool want_v = MODE == MODE_COMBINE && pv >= zs && pv < ze;
            const bool tma_u = want_u && !ghost_plane;
            LSG_CHECK(j >= 0 && j < NB && vj >= 0 && vj < NV && sj >= 0 && sj < NS);
            LSG_CHECK(!tma_u || (src + P.halo * W >= 0 && src + P.halo * W < P.n[2] + 2 * P.halo * W));
            LSG_CHECK(!want_v || (pv >= 0 && pv < P.n[2]));
            mbar_arrive_expect_tx(bar + j, (tma_u ? static_cast<unsigned>(pitch * (M.R + 2 * W) * 8) : 0u) +
                                               (want_v ? static_cast<unsigned>(TX * M.R * 8) : 0u));
            if (tma_u) tma_load_3d(ring + j * slot, &tmu, bar + j, x0 - XL, y0 - W, src + P.halo * W);
            if (want_v) tma_load_3d(vring + vj * M.vslot, &tmv, bar + j, x0, y0, pv + P.halo * W);
        }
        if (!generic_writes || !want_u) return;
        double* buf = ring + j * slot;
        if (ghost_plane) {
            // extrapolated plane beyond a global boundary (grid.cpp:120-126): plain loads
            const int e0 = zg < 0 ? 0 : nglob - 1, e1 = zg < 0 ? 1 : nglob - 2;
            const double k = (double)(zg < 0 ? -zg : zg - (nglob - 1));
            const double* b0 = P.u + (long long)(e0 - P.z0) * s2;
            const double* b1 = P.u + (long long)(e1 - P.z0) * s2;
            LSG_CHECK(e0 - P.z0 >= -P.halo * W && e0 - P.z0 < P.n[2] + P.halo * W);
            LSG_CHECK(e1 - P.z0 >= -P.halo * W && e1 - P.z0 < P.n[2] + P.halo * W);
            auto ext = [&](int o) {
                const double lo = __ldg(b0 + o);
                return lo + k * (lo - __ldg(b1 + o));
            };
            if (active) buf[me] = ext(coli);
            if (two) buf[me + 1] = ext(coli + 1);
            for (int h = t; h < nh; h += blockDim.x) {
                int off, gx, gy;
                const bool out = halo_cell(h, off, gx, gy);
                const bool wx = gx < 0 || gx >= n0, wy = gy < 0 || gy >= n1;
                if (out && ((wx && P.bc[0] != LSG_BC_PERIODIC) || (wy && P.bc[1] != LSG_BC_PERIODIC))) continue;
                gx = gx < 0 ? gx + n0 : (gx >= n0 ? gx - n0 : gx);
                gy = gy < 0 ? gy + n1 : (gy >= n1 ? gy - n1 : gy);
                buf[off] = ext(gy * n0 + gx);
            }
        } else if (border) {
            // periodic wraps: cp.async into the staging slot (copied in after the TMA lands)
            const double* base = P.u + (long long)src * s2;
            LSG_CHECK(src >= -P.halo * W && src < P.n[2] + P.halo * W);
#pragma unroll
            for (int q = 0; q < kMaxHalo; ++q)
                if (c_off[q] >= 0 && c_b[q] < 0) cp_async8(stage + sj * M.hmax + t + q * blockDim.x, base + c_a[q]);
        }
    };
    // Plane p landed in u slot j (every thread waits on the slot's mbarrier):
    // fix the border tile's out-of-range halo cells (this thread's own wrap
    // copies after its cp.async group completes; extrapolated ghosts in place).
    auto fixup = [&](int p, int j, int sj) {
        if (!border || p >= ze + W) return;
        double* buf = ring + j * slot;
        const int zg = P.z0 + p;
        const bool ghost_plane = (zg < 0 || zg >= nglob) && P.bc[2] != LSG_BC_PERIODIC;
#pragma unroll
        for (int q = 0; q < kMaxHalo; ++q) {
            if (c_off[q] < 0) continue;
            if (c_b[q] < 0) {  // periodic wrap
                if (!ghost_plane) buf[c_off[q]] = stage[sj * M.hmax + t + q * blockDim.x];
            } else {  // dst[w-k] = lo + k*(lo - x1), dst[w+n-1+k] = hi + k*(hi - x_{n-2})
                const double a = buf[c_a[q]];
                buf[c_off[q]] = a + (double)(c_b[q] >> 24) * (a - buf[c_b[q] & 0xFFFFFF]);
            }
        }
    };

    asm volatile("griddepcontrol.wait;\n" ::: "memory");

    // ---- prologue: u-planes zs-W .. zs+W+D-1 in flight (slots 0..2W+D-1),
    // the first 2W landed and fixed (staging holds D + 1 planes, so each is
    // fixed once D newer ones are in flight)
#pragma unroll 1
    for (int k = 0; k < 2 * W + D; ++k) {
        issue(zs - W + k, k, k >= 2 * W ? k - 2 * W : 0, k % NS);  // v0-plane zs-2W+k (from k = 2W) in slot k-2W
        if (generic_writes) cp_async_commit();
        if (k >= D) {
            if (generic_writes) {
                cp_async_wait<D>();
                __syncthreads();  // extrapolated planes written by other threads
            }
            mbar_wait(bar + (k - D), 0u);
            fixup(zs - W + k - D, k - D, (k - D) % NS);
        }
    }

    if constexpr (YP) {
        __syncthreads();              // plane zs (slot W) fixed by every thread
        ypass(ring + W * slot, ybuf);  // its y terms, read at z = zs
    }

    unsigned long long kmin = ~0ull, kmax = 0ull;
    unsigned fz = ~0u;
    bool bad = false;
    const double ax0 = __ldg(P.axis[0] + x), ax1 = __ldg(P.axis[0] + x + (two ? 1 : 0));
    const double ay = __ldg(P.axis[1] + y);
    double az = __ldg(P.axis[2] + P.z0 + zs);
    Trig tr = load_trig<KIND>(P, P.z0 + zs, 0);

    // Ring bookkeeping, one plane per iteration: u slot j0 holds plane z-W, so
    // plane z+W sits in j0+2W and plane z+W+D goes into j0-1 (mod NB, the slot
    // plane z-W-1 has just left); v0 slot vr holds plane z, plane z+D goes into
    // vr-1 (mod NV).  Each u slot's mbarrier completes once per use: the parity
    // of plane z+W's wait flips every time its slot index wraps.
    Eno3Z qa, qb;  // ENO3: z tables of the pair carried along the march
    int j0 = 0, vr = 0, sr = (2 * W) % NS;  // staging slot of plane z+W
    unsigned par = 0u;                      // parity bit per u slot (planes zs-W..zs+W-1 consumed once)
#pragma unroll
    for (int k = 0; k < 2 * W; ++k) par ^= 1u << k;
#pragma unroll 1
    for (int z = zs; z < ze; ++z) {
        const int jw = j0 + 2 * W >= NB ? j0 + 2 * W - NB : j0 + 2 * W;  // plane z+W
        const bool zeven = ((z - zs) & 1) == 0;
        if (generic_writes) cp_async_wait<D - 1>();  // this thread's wrap copies of plane z+W
        if (!ZP || zeven) {
            mbar_wait(bar + jw, (par >> jw) & 1u);
            par ^= 1u << jw;
        }
        // plane z+W+1 for the z lines of plane z+1 (own cells only: no fix-up
        // needed).  An odd chunk's last plane has no plane z+1: node b of its
        // z lines reads a stale slot, and node a's bits do not depend on it
        // (line_lr2: a's window is s[0..2W]; an operand outside the fast
        // divisions' domain only sends both to the IEEE path)
        if (ZP && zeven && z + 1 < ze) {
            const int jn = jw + 1 == NB ? 0 : jw + 1;
            mbar_wait(bar + jn, (par >> jn) & 1u);
            par ^= 1u << jn;
        }
        fixup(z + W, jw, sr);
        // generic-proxy writes of the ring (fix-ups, extrapolated planes) before
        // the TMA writes that will reuse their slots (issued after the barrier)
        if (generic_writes) asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
        __syncthreads();  // fix-ups visible; the slot of plane z-W-1 is free
        {
            const int ji = j0 == 0 ? NB - 1 : j0 - 1;
            const int vi = vr == 0 ? NV - 1 : vr - 1;
            const int si = sr + D >= NS ? sr + D - NS : sr + D;
            issue(z + W + D, ji, vi, si);
            if (generic_writes) cp_async_commit();
        }
        const double* zpl[2 * W + 2];
#pragma unroll
        for (int k = 0; k < 2 * W + 2; ++k) {
            const int j = j0 + k;
            zpl[k] = ring + (j >= NB ? j - NB : j) * slot + me;
        }
        double azn = 0.0;
        Trig trn;
        if (z + 1 < ze) {
            azn = __ldg(P.axis[2] + P.z0 + z + 1);
            trn = load_trig<KIND>(P, P.z0 + z + 1, 0);
        }
        // y terms of plane z+1 (resident: z+1 <= z+W) into the other buffer; the
        // pairs of plane z-1 read it before this iteration's barrier
        const int yp = (z - zs) & 1;
        if (YP && z + 1 < ze) {
            const int j = j0 + W + 1;
            ypass(ring + (j >= NB ? j - NB : j) * slot, ybuf + (yp ^ 1) * TX * M.R);
        }
        if (active)
            march3_pair<S, KIND, MODE, RANGE, S == ENO3, YP, ZP>(
                P, zpl, me, pitch, MODE == MODE_COMBINE ? vring + vr * M.vslot + vme : nullptr, coli, z, two, ax0,
                ax1, ay, az, tr, kmin, kmax, fz, bad, &qa, &qb, z == zs, ybuf + yp * TX * M.R + vme, zst, zeven);
        az = azn;
        tr = trn;
        j0 = j0 + 1 == NB ? 0 : j0 + 1;
        vr = vr + 1 == NV ? 0 : vr + 1;
        sr = sr + 1 == NS ? 0 : sr + 1;
    }
    if (generic_writes) cp_async_wait<0>();
    asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");

    if (P.flags && __any_sync(0xffffffffu, bad) && (t & 31) == 0) atomicOr(P.flags, FLAG_HAM_NONFINITE);
    if (RANGE && P.range) block_range(P.range, kmin, kmax, fz == ~0u ? ~0ull : (unsigned long long)fz);
}

using March3TmaFn = void (*)(StageParams, March3, CUtensorMap, CUtensorMap);

}  // namespace lsg
