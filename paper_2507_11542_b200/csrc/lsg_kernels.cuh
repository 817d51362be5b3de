// lsg_kernels.cuh — kernel templates of the HJ hot path.
//
//   stage_kernel   fused ghost fill + upwind L/R per dimension + central costate +
//                  Hamiltonian + global-LF dissipation + clamp + TVD-RK stage
//                  combination (+ v range for the step log); nothing but the
//                  stage output is written to HBM.  Replaces the reference's
//                  ~3D+4 full-field passes per term (hamiltonian.cpp:11-76) and
//                  the RK loops (integrator.cpp:58-92).
//   alpha_kernel   per-dimension max of the dissipation bound: warp shuffle ->
//                  block (smem) -> one 64-bit atomicMax per block on the bit
//                  pattern of the non-negative double (exact, order-free).
//
// Generic over the grid dimension D (1..6): one thread per node, the
// cross-shaped stencil read through the read-only data path (neighbouring
// threads share lines through L1/L2).  3-D grids take the 2.5-D tiled
// kernel in lsg_march3.cuh; this one serves D != 3, the gapped boundary-band
// launches of slabs, and LSG_KERNEL=generic.
#pragma once

#include "lsg_device.cuh"

namespace lsg {

using StageFn = void (*)(StageParams);

// Warp maximum of a 64-bit key: two 32-bit redux.sync (the maximum's high
// word, then the largest low word among the lanes holding it).  Every lane
// of the warp must call it.
__device__ __forceinline__ unsigned long long warp_max_u64(unsigned long long x) {
    const unsigned hi = static_cast<unsigned>(x >> 32), lo = static_cast<unsigned>(x);
    const unsigned mhi = __reduce_max_sync(0xffffffffu, hi);
    const unsigned mlo = __reduce_max_sync(0xffffffffu, hi == mhi ? lo : 0u);
    return (static_cast<unsigned long long>(mhi) << 32) | mlo;
}

// Block reduction of a step's range candidates into its slot:
// {~min key, max key, ~first zero code} (all max-reduced, also across ranks).
// Every thread of the block must call it.
__device__ __forceinline__ void block_range(unsigned long long* slot, unsigned long long kmin, unsigned long long kmax,
                                            unsigned long long fz) {
    unsigned long long nmin = warp_max_u64(~kmin), mx = warp_max_u64(kmax), nfz = warp_max_u64(~fz);
    __shared__ unsigned long long smin[32], smax[32], sfz[32];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (lane == 0) {
        smin[warp] = nmin;
        smax[warp] = mx;
        sfz[warp] = nfz;
    }
    __syncthreads();
    if (warp == 0) {
        const int nw = blockDim.x >> 5;
        nmin = warp_max_u64(lane < nw ? smin[lane] : 0ull);
        mx = warp_max_u64(lane < nw ? smax[lane] : 0ull);
        nfz = warp_max_u64(lane < nw ? sfz[lane] : 0ull);
        if (lane == 0) {
            if (nmin) atomicMax(slot, nmin);
            if (mx) atomicMax(slot + 1, mx);
            if (nfz) atomicMax(slot + 2, nfz);
        }
    }
}

// One node's line as an out-of-line call: the 6-D exact-WENO5 kernel calls it
// once per dimension, so one copy of the scheme's code serves all six
// (unrolled, they overflow the instruction cache) while the dimension loop
// stays unrolled (p[] in registers).  Measured (41^6 / 81^4): exact WENO5
// 9.40 -> 9.63 G in 6-D, but 15.64 -> 15.10 G in 4-D; the fast WENO5 (18.7 ->
// 17.4 G) and ENO3 (21.8 -> 19.1 G) lose in 6-D, so exact WENO5 in 6-D only.
struct LRv {
    double L, R;
};
template <int S>
static __device__ __noinline__ LRv line_call(double s0, double s1, double s2, double s3, double s4, double s5,
                                             double s6, LineConst c) {
    const double s[7] = {s0, s1, s2, s3, s4, s5, s6};
    LRv r;
    line_lr<S>(s, c, r.L, r.R);
    return r;
}
template <int S, int D>
struct OutOfLineLine {
    static constexpr bool value = D >= 6 && S == WENO5;
};

// One node of a fused stage (hamiltonian.cpp:11-88 + integrator.cpp:58-85):
// L/R per dimension, central costate, H, global-LF dissipation, clamp, and
// the TVD-RK combination of MODE.  Returns the stage output at idx.
template <int D, int S, int KIND, int MODE>
__device__ __forceinline__ double stage_node(const StageParams& P, const double* u, const double* v0, double dt,
                                             double c, long long idx, bool& bad) {
    constexpr int W = SchemeWidth<S>::W;
    int i[D], ix[D];
    double x[D];
    long long r = idx;
#pragma unroll
    for (int d = 0; d < D; ++d) {
        if (d == D - 1) {
            i[d] = (int)r;
        } else {
            if (P.div31 & (d == 0 ? 1 : 2))
                r = divmod31(static_cast<unsigned>(r), P.n[d], P.magic[d], P.mshift[d], i[d]);
            else
                r = divmod_index(r, P.n[d], P.inv_n[d], i[d]);
        }
        ix[d] = (d == D - 1) ? P.z0 + i[d] : i[d];
        x[d] = __ldg(P.axis[d] + ix[d]);
    }
    double p[D];
    double diss = 0.0;
#pragma unroll
    for (int d = 0; d < D; ++d) {
        double s[2 * W + 1];
        gather_window<W>(u, idx, i[d], P.n[d], P.stride[d], P.bc[d], d == D - 1, P.z0, P.nz_glob, P.halo, s,
                         -(long long)P.halo * W * P.plane, P.n_local + (long long)P.halo * W * P.plane);
        double L, R;
        if constexpr (OutOfLineLine<S, D>::value) {
            const LRv r = line_call<S>(s[0], s[1], s[2], s[3], s[4], s[5], s[6], P.lc[d]);
            L = r.L;
            R = r.R;
        } else {
            line_lr<S>(s, P.lc[d], L, R);
        }
        costate<S>(P, d, L, R, p[d], diss);  // hamiltonian.cpp:31-32, 60-64
    }
    const double H = hamiltonian<KIND, D>(P, x, load_trig<KIND>(P, D > 2 ? ix[D > 2 ? 2 : 0] : 0, D > 5 ? ix[D > 5 ? 5 : 0] : 0), p);
    bad |= !isfinite(H);                    // hamiltonian.cpp:38-40
    double dv = -(H - 0.5 * diss);          // hamiltonian.cpp:65
    if (P.restrict_update)                  // hamiltonian.cpp:78-88
        dv = P.direction == LSG_GROW ? ((0.0 < dv) ? 0.0 : dv) : ((dv < 0.0) ? 0.0 : dv);
    if constexpr (MODE == MODE_TERM) {
        return dv;
    } else if constexpr (MODE == MODE_EULER) {
        return __ldg(u + idx) + dt * dv;
    } else {
        const double base = v0[idx];  // plain load: out may alias v0 (in-place RK update)
        return base + c * ((__ldg(u + idx) + dt * dv) - base);
    }
}

template <int D, int S, int KIND, int MODE>
__global__ void __launch_bounds__(256, 4) stage_kernel(const __grid_constant__ StageParams P) {
    const long long lidx = (long long)P.zlo * P.plane + (long long)blockIdx.x * blockDim.x + threadIdx.x;
    const long long idx = lidx >= (long long)P.zsplit * P.plane ? lidx + (long long)P.zskip * P.plane : lidx;
    unsigned long long kmin = ~0ull, kmax = 0ull, fz = ~0ull;
    bool bad = false;
    asm volatile("griddepcontrol.wait;\n" ::: "memory");  // programmatic dependent launch
    if (lidx < (long long)P.zhi * P.plane) {
        const double o = stage_node<D, S, KIND, MODE>(P, P.u, P.v0, P.dt, P.c, idx, bad);
        P.out[idx] = o;
        kmin = kmax = order_key(o);
        fz = zero_code(o, (unsigned long long)((long long)P.z0 * P.plane + idx));
    }
    asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");
    if (P.flags) {
        if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) atomicOr(P.flags, FLAG_HAM_NONFINITE);
    }
    if (P.range) {
        block_range(P.range, kmin, kmax, fz);
    }
}

// Parameters of the alpha reduction.
struct AlphaParams {
    long long n_local;
    int D;
    int n[kMaxDim];
    int z0;
    const double* axis[kMaxDim];
    const double* tcos[kMaxDim];
    const double* tsin[kMaxDim];
    int trig_dim;  // axis whose cos/sin the bound uses (-1: none)
    double hp[LSG_MAX_PARAMS];
    unsigned long long* out;  // D keys (bit patterns of non-negative doubles)
    unsigned* flags;
};

template <int KIND>
__global__ void __launch_bounds__(256) alpha_kernel(const __grid_constant__ AlphaParams A) {
    const long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    double x[kMaxDim] = {0, 0, 0, 0, 0, 0};
    double ct = 0.0, sn = 0.0;
    const bool live = idx < A.n_local;
    if (live) {
        long long r = idx;
        for (int d = 0; d < A.D; ++d) {
            int id;
            if (d == A.D - 1) {
                id = (int)r + A.z0;
            } else {
                const long long q = r / A.n[d];
                id = (int)(r - q * A.n[d]);
                r = q;
            }
            x[d] = A.axis[d][id];
            if (d == A.trig_dim) {
                ct = A.tcos[d][id];
                sn = A.tsin[d][id];
            }
        }
    }
    __shared__ unsigned long long sm[kMaxDim][8];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    bool bad = false;
    for (int d = 0; d < A.D; ++d) {
        unsigned long long key = 0ull;
        if (live) {
            double b = dissipation_bound<KIND>(A.hp, d, x, ct, sn);
            if (!isfinite(b) || b < 0.0) {  // hamiltonian.cpp:49-53
                bad = true;
                b = 0.0;
            }
            if (b == 0.0) b = 0.0;  // -0.0 -> +0.0: std::max(0.0, -0.0) keeps +0.0
            key = (unsigned long long)__double_as_longlong(b);
        }
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) key = max(key, __shfl_xor_sync(0xffffffffu, key, off));
        if (lane == 0) sm[d][warp] = key;
    }
    if (__any_sync(0xffffffffu, bad) && lane == 0) atomicOr(A.flags, FLAG_BOUND_INVALID);
    __syncthreads();
    if (warp == 0) {
        const int nw = blockDim.x >> 5;
        for (int d = 0; d < A.D; ++d) {
            unsigned long long key = lane < nw ? sm[d][lane] : 0ull;
#pragma unroll
            for (int off = 4; off > 0; off >>= 1) key = max(key, __shfl_xor_sync(0xffffffffu, key, off));
            if (lane == 0 && key) atomicMax(A.out + d, key);
        }
    }
}

// The device Hamiltonian / dissipation bound as the reference's plugins
// compute them (HamiltonianFn / DissipationFn, hamiltonian.hpp:16-25): H at
// every node from D costate fields, or the bound of dimension `dim`; raw
// values, no validation (term_lax_friedrichs validates).
struct EvalParams {
    StageParams P;                  // geometry, coordinate / trig tables, Hamiltonian parameters
    const double* costate[kMaxDim];
    int dim;                        // -1: Hamiltonian, else the dissipation bound of this dimension
    double* out;
};

template <int KIND, int D>
__global__ void __launch_bounds__(256) eval_kernel(const __grid_constant__ EvalParams E) {
    const long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (idx >= E.P.n_local) return;
    int ix[D];
    double x[kMaxDim] = {0, 0, 0, 0, 0, 0};
    long long r = idx;
#pragma unroll
    for (int d = 0; d < D; ++d) {
        int i;
        if (d == D - 1) {
            i = (int)r;
        } else {
            r = divmod_index(r, E.P.n[d], E.P.inv_n[d], i);
        }
        ix[d] = (d == D - 1) ? E.P.z0 + i : i;
        x[d] = __ldg(E.P.axis[d] + ix[d]);
    }
    const Trig tr = load_trig<KIND>(E.P, D > 2 ? ix[D > 2 ? 2 : 0] : 0, D > 5 ? ix[D > 5 ? 5 : 0] : 0);
    if (E.dim < 0) {
        double p[D];
#pragma unroll
        for (int d = 0; d < D; ++d) p[d] = __ldg(E.costate[d] + idx);
        E.out[idx] = hamiltonian<KIND, D>(E.P, x, tr, p);
    } else {
        E.out[idx] = dissipation_bound<KIND>(E.P.hp, E.dim, x, tr.c2, tr.s2);
    }
}

using EvalFn = void (*)(EvalParams);

}  // namespace lsg
