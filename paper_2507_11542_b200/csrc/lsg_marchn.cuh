// lsg_marchn.cuh — tile-and-march stage kernel for 4-D..6-D grids (sm_100a).
//
// The 3-D kernel's scheme applied to the first three axes of a D-dimensional
// grid: a block takes a TX x R tile of the (x, y) plane at one index of the
// outer axes 3..D-1 and marches along z (axis 2) through a balanced chunk of
// planes, with the x/y/z windows from a shared-memory ring of (x, y) planes
// whose halo cells hold the padded-line values (cp.async, ghost fill in
// shared memory, as march3_kernel; the rows of the 4-D/6-D configs are odd,
// 81 and 41 doubles, so not TMA-fed).  The outer axes' windows are read
// through the read-only path (L1/L2) with gather_window, the slab axis (the
// last one) with its halo planes.  Versus the one-thread-per-node kernel:
// three of the D windows need no per-node index arithmetic or ghost
// branches, the pair of x-adjacent nodes shares its x window and (WENO5) its
// constant quotients, and the index decomposition is per block.  Same
// arithmetic per node (line_lr, hamiltonian, finish), hence the same bits.
#pragma once

#include "lsg_march3.cuh"

namespace lsg {

// Node-pair update for D > 3: x/y/z from the shared windows (as march3_pair),
// axes 3..D-1 from global memory; writes the outputs, returns range candidates.
template <int D, int S, int KIND, int MODE, bool RANGE>
__device__ __forceinline__ void marchn_pair(const StageParams& P, const double* const* zpl, int me, int pitch,
                                            const double* vpair, long long idx, const int* io, int z, bool two,
                                            const double* xs_base, double ax1, const Trig& tr,
                                            unsigned long long& kmin, unsigned long long& kmax,
                                            unsigned long long& fz, bool& bad) {
    constexpr int W = SchemeWidth<S>::W;
    using RS = RingShape<W>;
    constexpr int SH = RS::SH, XW = RS::XW;
    const double* cur = zpl[W] - me;
    double L, R;
    double pa[D], pb[D];
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
        costate<S>(P, 0, L, R, pa[0], da);
        costate<S>(P, 0, L2, R2, pb[0], db);
    }
    double ca, cb;
    {   // y
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
        costate<S>(P, 1, L, R, pa[1], da);
        line_lr<S>(wb, P.lc[1], L, R);
        costate<S>(P, 1, L, R, pb[1], db);
    }
    {   // z
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
    }
    const long long lo = -(long long)P.halo * W * P.plane, hi = P.n_local + (long long)P.halo * W * P.plane;
#pragma unroll
    for (int d = 3; d < D; ++d) {  // outer axes: windows through L1/L2 (grid.cpp:108-128 ghost rules)
        double s[2 * W + 1];
        gather_window<W>(P.u, idx, io[d], P.n[d], P.stride[d], P.bc[d], d == D - 1, P.z0, P.nz_glob, P.halo, s, lo,
                         hi);
        line_lr<S>(s, P.lc[d], L, R);
        costate<S>(P, d, L, R, pa[d], da);
        if (two) {
            gather_window<W>(P.u, idx + 1, io[d], P.n[d], P.stride[d], P.bc[d], d == D - 1, P.z0, P.nz_glob, P.halo,
                             s, lo, hi);
            line_lr<S>(s, P.lc[d], L, R);
        }
        costate<S>(P, d, L, R, pb[d], db);
    }
    double b0 = 0.0, b1 = 0.0;
    if (MODE == MODE_COMBINE) {
        const double2 v = *reinterpret_cast<const double2*>(vpair);
        b0 = v.x;
        b1 = v.y;
    }
    double xs[D];
#pragma unroll
    for (int d = 0; d < D; ++d) xs[d] = xs_base[d];
    auto finish = [&](const double* p, double diss, double centre, double base, bool& b) {
        const double H = hamiltonian<KIND, D>(P, xs, tr, p);
        b |= !isfinite(H);
        double dv = -(H - 0.5 * diss);
        if (P.restrict_update) dv = P.direction == LSG_GROW ? ((0.0 < dv) ? 0.0 : dv) : ((dv < 0.0) ? 0.0 : dv);
        if constexpr (MODE == MODE_TERM) return dv;
        else if constexpr (MODE == MODE_EULER) return centre + P.dt * dv;
        else return base + P.c * ((centre + P.dt * dv) - base);
    };
    const double oa = finish(pa, da, ca, b0, bad);
    xs[0] = ax1;
    bool bad_b = false;
    const double ob = finish(pb, db, cb, b1, bad_b);
    LSG_CHECK(idx >= 0 && idx + (two ? 1 : 0) < P.n_local);
    P.out[idx] = oa;
    if (two) {
        P.out[idx + 1] = ob;
        bad |= bad_b;
    }
    if (RANGE) {
        const unsigned long long ka = order_key(oa), kb = two ? order_key(ob) : ka;
        kmin = min(kmin, min(ka, kb));
        kmax = max(kmax, max(ka, kb));
        if (oa == 0.0 || (two && ob == 0.0)) {
            const unsigned long long g = (unsigned long long)((long long)P.z0 * P.plane + idx);
            const unsigned long long ca2 = zero_code(oa, g), cb2 = two ? zero_code(ob, g + 1) : ~0ull;
            fz = min(fz, min(ca2, cb2));
        }
    }
    (void)z;
}

// Grid: blockIdx.x = tile + ntiles * outer, outer = the block's index over the
// axes 3..D-1 (the last one over the launch's logical plane range, with the
// band gap); blockIdx.y = z-chunk.  Axis 2 is marched over its whole extent.
template <int D, int S, int KIND, int MODE, bool RANGE>
__global__ void __launch_bounds__(256, S <= ENO2 ? 3 : 2) marchn_kernel(const __grid_constant__ StageParams P,
                                                                       const __grid_constant__ March3 M) {
    constexpr int W = SchemeWidth<S>::W;
    using RS = RingShape<W>;
    constexpr int DD = RS::D, NB = RS::NB, NV = RS::NV, SH = RS::SH;
    extern __shared__ __align__(16) double sm[];
    const int n0 = P.n[0], n1 = P.n[1], n2 = P.n[2];
    const long long s2 = P.stride[2];
    const int TX = M.TX, pitch = M.pitch, TX2 = M.TX >> 1;
    const int plane_sz = pitch * (M.R + 2 * W);
    const int vplane_sz = TX * M.R;
    double* const ring = sm;
    double* const vring = sm + NB * plane_sz;
    const int t = threadIdx.x;
    const int ntiles = M.ntx * ((n1 + M.R - 1) / M.R);
    const int tile = blockIdx.x % ntiles;
    int outer = blockIdx.x / ntiles;
    const int xt = tile % M.ntx, yt = tile / M.ntx;
    const int x0 = xt * TX, y0 = yt * M.R;
    const int cols = min(TX, n0 - x0), rows = min(M.R, n1 - y0);
    // outer indices (local to the slab for the last axis)
    int io[D];
    long long obase = 0;
#pragma unroll
    for (int d = 3; d < D - 1; ++d) {
        io[d] = outer % P.n[d];
        outer /= P.n[d];
        obase += (long long)io[d] * P.stride[d];
    }
    {
        const int lz = P.zlo + outer;  // logical plane of the last axis
        io[D - 1] = lz >= P.zsplit ? lz + P.zskip : lz;
        obase += (long long)io[D - 1] * P.stride[D - 1];
    }
    const double* const u = P.u + obase;
    // z-chunk [zs, ze) of axis 2 (balanced split, longer chunks first)
    const int cbz = n2 / M.nzc, crem = n2 - cbz * M.nzc;
    const int cidx = blockIdx.y;
    const int zs = cidx * cbz + min(cidx, crem);
    const int ze = zs + cbz + (cidx < crem ? 1 : 0);
    const int yl = t / TX2, pl = t - (t / TX2) * TX2;
    const int xl = 2 * pl;
    const bool active = yl < rows && xl < cols;
    const bool two = active && xl + 1 < cols;
    const int x = x0 + (active ? xl : 0), y = y0 + (active ? yl : 0);
    const int coli = y * n0 + x;
    const int me = (yl + W) * pitch + (xl + W + SH);
    const int vme = yl * TX + xl;

    // ---- halo slots (x/y): copies from global, or ghosts computed in shared memory
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
                } else {
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

    const int ring_sz = NB * plane_sz, vring_sz = NV * vplane_sz;
    int is_off = 0, vi_off = 0, gp_off = 0;
    auto bump = [](int& off, int step, int size) {
        off += step;
        if (off == size) off = 0;
    };
    bool has_ghost = false;
#pragma unroll
    for (int q = 0; q < kMaxHalo; ++q) has_ghost |= hdst[q] >= 0 && hsrc[q] < 0;

    // u-plane p of axis 2 (window [zs-W, ze+W)) and v0-plane p-W
    auto issue = [&](int p) {
        if (p < ze + W) {
            double* buf = ring + is_off;
            int src = p;
            bool ghost_plane = false;
            if (p < 0 || p >= n2) {
                if (P.bc[2] == LSG_BC_PERIODIC) src = p < 0 ? p + n2 : p - n2;
                else ghost_plane = true;
            }
            if (!ghost_plane) {
                const double* base = u + (long long)src * s2;
                if (active) cp_async8(buf + me, base + coli);
                if (two) cp_async8(buf + me + 1, base + coli + 1);
#pragma unroll
                for (int q = 0; q < kMaxHalo; ++q)
                    if (hsrc[q] >= 0) cp_async8(buf + hdst[q], base + hsrc[q]);
            } else {  // grid.cpp:120-126
                const int e0 = p < 0 ? 0 : n2 - 1, e1 = p < 0 ? 1 : n2 - 2;
                const double k = (double)(p < 0 ? -p : p - (n2 - 1));
                const double* b0 = u + (long long)e0 * s2;
                const double* b1 = u + (long long)e1 * s2;
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
                const double* base = P.v0 + obase + (long long)pv * s2;
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

    asm volatile("griddepcontrol.wait;\n" ::: "memory");

#pragma unroll 1
    for (int p = zs - W; p < zs + W + DD; ++p) issue(p);
    cp_async_wait<DD>();
    __syncthreads();
#pragma unroll 1
    for (int p = zs - W; p < zs + W; ++p) ghost_pass(p);

    unsigned long long kmin = ~0ull, kmax = 0ull, fz = ~0ull;
    bool bad = false;
    // coordinates: x (two nodes), y, z per plane, outer axes per block; trig of
    // the heading axes 2 and 5 where the kind has them
    double xs[D];
    xs[0] = __ldg(P.axis[0] + x);
    const double ax1 = __ldg(P.axis[0] + x + (two ? 1 : 0));
    xs[1] = __ldg(P.axis[1] + y);
#pragma unroll
    for (int d = 3; d < D; ++d) xs[d] = __ldg(P.axis[d] + (d == D - 1 ? P.z0 + io[d] : io[d]));
    const int i5 = D > 5 ? (5 == D - 1 ? P.z0 + io[D > 5 ? 5 : 3] : io[D > 5 ? 5 : 3]) : 0;
    io[0] = x, io[1] = y;

    int j0 = 0, vr_off = 0;
#pragma unroll 1
    for (int z = zs; z < ze; ++z) {
        cp_async_wait<DD - 1>();
        __syncthreads();
        ghost_pass(z + W);
        issue(z + W + DD);
        const double* zpl[2 * W + 1];
#pragma unroll
        for (int k = 0; k < 2 * W + 1; ++k) {
            const int j = j0 + k;
            zpl[k] = ring + (j >= NB ? j - NB : j) * plane_sz + me;
        }
        j0 = j0 + 1 == NB ? 0 : j0 + 1;
        if (active) {
            xs[2] = __ldg(P.axis[2] + z);
            io[2] = z;
            const Trig tr = load_trig<KIND>(P, z, i5);
            const long long idx = obase + (long long)z * s2 + coli;
            marchn_pair<D, S, KIND, MODE, RANGE>(P, zpl, me, pitch,
                                                 MODE == MODE_COMBINE ? vring + vr_off + vme : nullptr, idx, io, z,
                                                 two, xs, ax1, tr, kmin, kmax, fz, bad);
        }
        bump(vr_off, vplane_sz, vring_sz);
    }
    cp_async_wait<0>();
    asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");

    if (P.flags && __any_sync(0xffffffffu, bad) && (t & 31) == 0) atomicOr(P.flags, FLAG_HAM_NONFINITE);
    if (RANGE && P.range) block_range(P.range, kmin, kmax, fz);
}

using MarchNFn = void (*)(StageParams, March3);

}  // namespace lsg
