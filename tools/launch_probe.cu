// tools/launch_probe.cu — floor costs at the bench size (1,030,301 nodes):
// empty kernel (small vs 1.5 KB __grid_constant__ param), a trivial 7-point
// stencil from L2, and the same with one same-address atomic per block.
#include <cstdio>
#include <cuda_runtime.h>

struct Big { double v[180]; const double* u; double* out; int n0, n1, nz; unsigned long long* r; };
struct Small { const double* u; double* out; int n0, n1, nz; unsigned long long* r; };

__global__ void empty_small(const __grid_constant__ Small p) {}
__global__ void empty_big(const __grid_constant__ Big p) {}

template <class PR, bool ATOM>
__global__ void __launch_bounds__(256) stencil(const __grid_constant__ PR p) {
    const int plane = p.n0 * p.n1;
    const int q = blockIdx.x * 256 + threadIdx.x;
    const int z = blockIdx.y;
    if (q >= plane) return;
    const int y = q / p.n0, x = q - y * p.n0;
    const long long i = (long long)z * plane + q;
    double s = p.u[i];
    if (x > 0 && x < p.n0 - 1 && y > 0 && y < p.n1 - 1 && z > 0 && z < p.nz - 1)
        s = (((s + p.u[i - 1]) + p.u[i + 1]) + (p.u[i - p.n0] + p.u[i + p.n0])) + (p.u[i - plane] + p.u[i + plane]);
    p.out[i] = s;
    if (ATOM && threadIdx.x == 0) atomicMax(p.r, (unsigned long long)__double_as_longlong(s));
}

template <class F>
float timeit(F f, int reps = 200) {
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    for (int i = 0; i < 10; ++i) f();
    cudaEventRecord(a);
    for (int i = 0; i < reps; ++i) f();
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    return ms / reps * 1e3f;
}

int main() {
    const int n = 101, N = n * n * n;
    double *u, *o;
    unsigned long long* r;
    cudaMalloc(&u, N * 8);
    cudaMalloc(&o, N * 8);
    cudaMalloc(&r, 8);
    cudaMemset(u, 0, N * 8);
    Small s{u, o, n, n, n, r};
    Big b{};
    b.u = u, b.out = o, b.n0 = n, b.n1 = n, b.nz = n, b.r = r;
    dim3 grid((n * n + 255) / 256, n);
    printf("empty small-param   %.2f us\n", timeit([&] { empty_small<<<1, 32>>>(s); }));
    printf("empty 1.5KB-param   %.2f us\n", timeit([&] { empty_big<<<1, 32>>>(b); }));
    printf("empty full grid     %.2f us\n", timeit([&] { empty_small<<<grid, 256>>>(s); }));
    printf("stencil small       %.2f us\n", timeit([&] { stencil<Small, false><<<grid, 256>>>(s); }));
    printf("stencil 1.5KB       %.2f us\n", timeit([&] { stencil<Big, false><<<grid, 256>>>(b); }));
    printf("stencil + atomic    %.2f us\n", timeit([&] { stencil<Small, true><<<grid, 256>>>(s); }));
    return 0;
}
