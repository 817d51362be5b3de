// tools/divfast_check.cu — div_fast (lsg_device.cuh), the branch-free replica
// of the compiler's IEEE double-division fast path, against `/` on 1e10
// inputs: numerators {0.1, 0.3, 0.6, 1} and random doubles, divisors
// log-uniform over [1e-12, 1e300] with random mantissas, plus divisors next to
// powers of two and to the numerators (ties and near-ties of the rounding).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "../paper_2507_11542_b200/csrc/lsg_device.cuh"

__device__ unsigned long long mix(unsigned long long z) {
    z += 0x9e3779b97f4a7c15ull;
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
    return z ^ (z >> 31);
}

__global__ void check(unsigned long long seed, long long n, unsigned long long* bad, double* ex) {
    const double nums[4] = {0.1, 0.3, 0.6, 1.0};
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
        const unsigned long long h = mix(seed + i), h2 = mix(h);
        // divisor: exponent uniform in [2^-39, 2^996] (~[1.8e-12, 6.7e299]), random mantissa
        const int e = -39 + (int)(h % 1036);
        unsigned long long bb = (h2 & 0x000FFFFFFFFFFFFFull) | ((unsigned long long)(e + 1023) << 52);
        if ((i & 7) == 0) bb = ((unsigned long long)(e + 1023) << 52) + (h2 & 3) - 1;  // next to a power of two
        double b = __longlong_as_double((long long)bb);
        double a = nums[(h >> 40) & 3];
        if ((i & 15) == 1) a = 1.0 + (double)(h2 >> 12) * 0x1p-52;  // random numerator in [1, 2)
        if ((i & 31) == 3) b = a * (1.0 + (double)((long long)(h2 & 7) - 3) * 0x1p-52);  // quotient near 1
        if (b < 1e-12 || b > 1e300) continue;
        const double q = lsg::div_fast(a, b), r = a / b;
        if (__double_as_longlong(q) != __double_as_longlong(r)) {
            if (atomicAdd(bad, 1ull) == 0) {
                ex[0] = a;
                ex[1] = b;
            }
        }
    }
}

int main() {
    unsigned long long* bad;
    double* ex;
    cudaMallocManaged(&bad, 8);
    cudaMallocManaged(&ex, 16);
    *bad = 0;
    const long long n = 1LL << 31;
    for (int rep = 0; rep < 5; ++rep) check<<<148 * 16, 256>>>(0xabcdefull + rep * n, n, bad, ex);
    cudaDeviceSynchronize();
    printf("checked %lld quotients: %llu mismatches%s\n", 5 * n, *bad, *bad ? "" : " (bit-exact)");
    if (*bad) printf("first mismatch: %a / %a\n", ex[0], ex[1]);
    return *bad ? 1 : 0;
}
