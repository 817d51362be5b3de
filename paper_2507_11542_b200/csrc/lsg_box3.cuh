// lsg_box3.cuh — one-node-per-thread fused stage kernel for 3-D grids.
//
// Block = 256 consecutive nodes of one z-plane's flattened (x, y) index, grid
// = (plane blocks, planes).  Interior nodes (every window inside the slab)
// read their three 2W+1 windows straight through the read-only path with
// constant strides; nodes near a domain edge take the ghost-rule gather
// (grid.cpp:108-128).  No tile pipeline, no barriers: latency is hidden by
// occupancy.  Arithmetic identical to stage_kernel (bit-exact).
#pragma once

#include "lsg_kernels.cuh"

namespace lsg {

template <int S, int KIND, int MODE, bool RANGE>
__global__ void __launch_bounds__(256) box3_kernel(const __grid_constant__ StageParams P) {
    constexpr int W = SchemeWidth<S>::W;
    const int n0 = P.n[0], n1 = P.n[1];
    const int plane = n0 * n1;
    const int q = blockIdx.x * 256 + threadIdx.x;
    const int zl = P.zlo + blockIdx.y;
    const int z = zl >= P.zsplit ? zl + P.zskip : zl;
    unsigned long long kmin = ~0ull, kmax = 0ull, fz = ~0ull;
    bool bad = false;
    if (q < plane) {
        const int y = q / n0, x = q - (q / n0) * n0;
        const long long idx = (long long)z * plane + q;
        const double* u = P.u + idx;
        const int zg = P.z0 + z;
        const bool zin = (zg >= W && zg < P.nz_glob - W) || (P.halo && P.bc[2] == LSG_BC_PERIODIC);
        double w0[2 * W + 1], w1[2 * W + 1], w2[2 * W + 1];
        if (x >= W && x < n0 - W && y >= W && y < n1 - W && zin) {
#pragma unroll
            for (int k = -W; k <= W; ++k) {
                w0[W + k] = __ldg(u + k);
                w1[W + k] = __ldg(u + k * n0);
                w2[W + k] = __ldg(u + (long long)k * plane);
            }
        } else {
            gather_window<W>(P.u, idx, x, n0, 1, P.bc[0], false, 0, n0, 0, w0);
            gather_window<W>(P.u, idx, y, n1, n0, P.bc[1], false, 0, n1, 0, w1);
            gather_window<W>(P.u, idx, z, P.n[2], plane, P.bc[2], true, P.z0, P.nz_glob, P.halo, w2);
        }
        double p[3];
        double diss = 0.0, L, R;
        line_lr<S>(w0, P.lc[0], L, R);
        costate<S>(P, 0, L, R, p[0], diss);
        line_lr<S>(w1, P.lc[1], L, R);
        costate<S>(P, 1, L, R, p[1], diss);
        line_lr<S>(w2, P.lc[2], L, R);
        costate<S>(P, 2, L, R, p[2], diss);
        const double xs[3] = {__ldg(P.axis[0] + x), __ldg(P.axis[1] + y), __ldg(P.axis[2] + zg)};
        const double H = hamiltonian<KIND, 3>(P, xs, load_trig<KIND>(P, zg, 0), p);
        bad = !isfinite(H);
        double dv = -(H - 0.5 * diss);
        if (P.restrict_update) dv = P.direction == LSG_GROW ? ((0.0 < dv) ? 0.0 : dv) : ((dv < 0.0) ? 0.0 : dv);
        double o;
        if constexpr (MODE == MODE_TERM) {
            o = dv;
        } else if constexpr (MODE == MODE_EULER) {
            o = w0[W] + P.dt * dv;
        } else {
            const double base = P.v0[idx];
            o = base + P.c * ((w0[W] + P.dt * dv) - base);
        }
        P.out[idx] = o;
        if (RANGE) {
            kmin = kmax = order_key(o);
            fz = zero_code(o, (unsigned long long)((long long)P.z0 * plane + idx));
        }
    }
    if (P.flags && __any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) atomicOr(P.flags, FLAG_HAM_NONFINITE);
    if (RANGE && P.range) block_range(P.range, kmin, kmax, fz);
}

using Box3Fn = void (*)(StageParams);

}  // namespace lsg
