// lsg_misc.cu — the non-fused kernels behind the reference-facing calls:
//   upwind_kernel   upwind_derivative for one dimension (spatial_derivatives.cpp:37-224)
//   pad_kernel      pad_ghost (grid.cpp:132-165)
//   shift_kernel    shift_along_dim (grid.cpp:167-193)
//   restrict_kernel restrict_update (hamiltonian.cpp:78-88)
//   shape_kernel    device initial conditions (implicit_surfaces.cpp:20-71)
//   range_init      step-log v range slots
#include "lsg_misc.cuh"

namespace lsg {

template <int S>
__global__ void __launch_bounds__(256) upwind_kernel(const __grid_constant__ StageParams P, int dim, int D,
                                                     double* __restrict__ left, double* __restrict__ right) {
    constexpr int W = SchemeWidth<S>::W;
    const long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (idx >= P.n_local) return;
    const int i = (int)((idx / P.stride[dim]) % P.n[dim]);
    double s[2 * W + 1];
    gather_window<W>(P.u, idx, i, P.n[dim], P.stride[dim], P.bc[dim], false, 0, P.n[dim], 0, s);
    double L, R;
    line_lr<S>(s, P.lc[dim], L, R);
    left[idx] = L;
    right[idx] = R;
    (void)D;
}

void launch_upwind(const StageParams& P, int dim, int D, int scheme, double* left, double* right,
                   cudaStream_t st) {
    const unsigned blocks = (unsigned)((P.n_local + 255) / 256);
    switch (scheme) {
        case FIRST: upwind_kernel<FIRST><<<blocks, 256, 0, st>>>(P, dim, D, left, right); break;
        case ENO2: upwind_kernel<ENO2><<<blocks, 256, 0, st>>>(P, dim, D, left, right); break;
        case ENO3: upwind_kernel<ENO3><<<blocks, 256, 0, st>>>(P, dim, D, left, right); break;
        default: upwind_kernel<WENO5><<<blocks, 256, 0, st>>>(P, dim, D, left, right); break;
    }
}

__global__ void __launch_bounds__(256) pad_kernel(const double* __restrict__ u, double* __restrict__ out,
                                                  long long n_out, int n, long long stride, int width, int bc) {
    const long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (idx >= n_out) return;
    const long long pblock = stride * (long long)(n + 2 * width);
    const long long outer = idx / pblock;
    const long long rem = idx - outer * pblock;
    const int j = (int)(rem / stride);
    const long long inner = rem - (long long)j * stride;
    const long long base = outer * stride * n + inner;
    const int jj = j - width;  // node index along the line
    double val;
    if (jj >= 0 && jj < n) {
        val = u[base + (long long)jj * stride];
    } else if (bc == LSG_BC_PERIODIC) {
        const int jw = jj < 0 ? jj + n : jj - n;
        val = u[base + (long long)jw * stride];
    } else if (jj < 0) {
        const double lo = u[base];
        const double ls = lo - u[base + stride];
        val = lo + (double)(-jj) * ls;
    } else {
        const double hi = u[base + (long long)(n - 1) * stride];
        const double hs = hi - u[base + (long long)(n - 2) * stride];
        val = hi + (double)(jj - (n - 1)) * hs;
    }
    out[idx] = val;
}

void launch_pad(const double* u, double* out, long long n_out, int n, long long stride, int width, int bc,
                cudaStream_t st) {
    pad_kernel<<<(unsigned)((n_out + 255) / 256), 256, 0, st>>>(u, out, n_out, n, stride, width, bc);
}

__global__ void __launch_bounds__(256) shift_kernel(const double* __restrict__ padded, double* __restrict__ out,
                                                    long long N, int n, long long stride, int width, int offset) {
    const long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (idx >= N) return;
    const long long lblock = stride * (long long)n;
    const long long outer = idx / lblock;
    const long long rem = idx - outer * lblock;
    const int j = (int)(rem / stride);
    const long long inner = rem - (long long)j * stride;
    out[idx] = padded[outer * stride * (long long)(n + 2 * width) + inner + (long long)(width + offset + j) * stride];
}

void launch_shift(const double* padded, double* out, long long N, int n, long long stride, int width, int offset,
                  cudaStream_t st) {
    shift_kernel<<<(unsigned)((N + 255) / 256), 256, 0, st>>>(padded, out, N, n, stride, width, offset);
}

__global__ void __launch_bounds__(256) restrict_kernel(const double* __restrict__ in, double* __restrict__ out,
                                                       long long n, int direction) {
    const long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (idx >= n) return;
    const double d = in[idx];
    out[idx] = direction == LSG_GROW ? ((0.0 < d) ? 0.0 : d) : ((d < 0.0) ? 0.0 : d);
}

void launch_restrict(const double* in, double* out, long long n, int direction, cudaStream_t st) {
    restrict_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(in, out, n, direction);
}

// Device initial conditions (implicit_surfaces.cpp:20-126), exact operation
// order: 0 sphere, 1 cylinder (:20-71), 2 planar pair distance |(x0,x1)-(x3,x4)|
// - r (cfg4 target set, builder-defined), 3 rectangle (:73-94), 4 ellipsoid
// (:96-116); composed with the resident field by op (set_union / set_intersection,
// :128-145: std::min / std::max of (field, shape)).
__device__ __forceinline__ double std_max(double a, double b) { return (a < b) ? b : a; }  // std::max
__device__ __forceinline__ double std_min(double a, double b) { return (b < a) ? b : a; }  // std::min

__global__ void __launch_bounds__(256) shape_kernel(const __grid_constant__ ShapeParams S) {
    const long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (idx >= S.n_local) return;
    double x[kMaxDim];
    long long r = idx;
    for (int d = 0; d < S.D; ++d) {
        int id;
        if (d == S.D - 1) {
            id = (int)r + S.z0;
        } else {
            const long long q = r / S.n[d];
            id = (int)(r - q * S.n[d]);
            r = q;
        }
        x[d] = S.axis[d][id];
    }
    double v;
    if (S.shape == 3) {
        v = -INFINITY;
        for (int d = 0; d < S.D; ++d) v = std_max(v, std_max(S.center[d] - x[d], x[d] - S.upper[d]));
    } else if (S.shape == 4) {
        v = x[0] * x[0] + 4.0 * x[1] * x[1];
        if (S.D == 3) v += 9.0 * x[2] * x[2];
        v = v - S.radius;
    } else {
        double r2 = 0.0;
        if (S.shape == 2) {
            const double a = x[0] - x[3];
            const double b = x[1] - x[4];
            r2 += a * a;
            r2 += b * b;
        } else {
            for (int d = 0; d < S.D; ++d) {
                if (S.ignored_mask & (1u << d)) continue;
                const double dx = x[d] - S.center[d];
                r2 += dx * dx;
            }
        }
        v = sqrt(r2) - S.radius;
    }
    if (S.op == 1) v = std_min(S.out[idx], v);
    else if (S.op == 2) v = std_max(S.out[idx], v);
    S.out[idx] = v;
}

void launch_shape(const ShapeParams& S, cudaStream_t st) {
    shape_kernel<<<(unsigned)((S.n_local + 255) / 256), 256, 0, st>>>(S);
}

__global__ void __launch_bounds__(256) set_op_kernel(int op, long long n, const double* __restrict__ a,
                                                     const double* __restrict__ b, double* __restrict__ out) {
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    out[i] = op == 1 ? std_min(a[i], b[i]) : (op == 2 ? std_max(a[i], b[i]) : -a[i]);
}

void launch_set_op(int op, long long n, const double* a, const double* b, double* out, cudaStream_t st) {
    set_op_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(op, n, a, b, out);
}

__global__ void range_init_kernel(unsigned long long* r, long long nslots) {
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < nslots) {
        r[2 * i] = ~0ull;
        r[2 * i + 1] = 0ull;
    }
}

void launch_range_init(unsigned long long* r, long long nslots, cudaStream_t st) {
    range_init_kernel<<<(unsigned)((nslots + 255) / 256), 256, 0, st>>>(r, nslots);
}

}  // namespace lsg

namespace lsg {
__global__ void stamp_kernel(unsigned long long* out) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    *out = t;
}
void launch_stamp(unsigned long long* out, cudaStream_t st) { stamp_kernel<<<1, 1, 0, st>>>(out); }
}  // namespace lsg

namespace lsg {
// FP64 issue-rate probe (the second roofline of the stencil, measured in the
// run that reports against it): 8 independent DADD/DMUL chains per thread,
// 8 blocks of 256 threads per SM; one op per chain and iteration (iters even).
__global__ void __launch_bounds__(256) fp64_rate_kernel(double* out, int iters, double a, double b) {
    double r[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) r[k] = threadIdx.x * 1e-3 + k;
    for (int i = 0; i < iters; i += 2) {
#pragma unroll
        for (int k = 0; k < 8; ++k) r[k] = __dadd_rn(r[k], a);
#pragma unroll
        for (int k = 0; k < 8; ++k) r[k] = __dmul_rn(r[k], b);
    }
    double s = 0.0;
#pragma unroll
    for (int k = 0; k < 8; ++k) s += r[k];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
void launch_fp64_rate(double* out, int blocks, int iters, cudaStream_t st) {
    fp64_rate_kernel<<<blocks, 256, 0, st>>>(out, iters, 1e-9, 1.0000001);
}
}  // namespace lsg
