// Exhaustive-style check of divmod_index (lsg_device.cuh), the per-node index
// decomposition of the generic stage kernel: against exact 64-bit integer
// division for x in [0, 2^40) and every divisor 1..65536, concentrated on
// the values next to multiples of d (where a quotient estimate off by one
// would show) plus uniform random x.  Prints "divmod ok <n>" or the first
// mismatch; built by __graft_entry__.build(), run by tests/test_gpu_shim.py.
#include <cstdio>
#include <cuda_runtime.h>

#include "../../paper_2507_11542_b200/csrc/lsg_device.cuh"

__device__ unsigned long long g_bad = 0, g_count = 0;
__device__ long long g_x = -1;
__device__ int g_d = 0;

__device__ __forceinline__ unsigned long long mix(unsigned long long z) {
    z += 0x9e3779b97f4a7c15ull;
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
    return z ^ (z >> 31);
}

__global__ void check(int dmax, int per_d) {
    const int d = 1 + blockIdx.x % dmax;
    const double inv = 1.0 / d;
    unsigned long long bad = 0, cnt = 0;
    for (int k = threadIdx.x; k < per_d; k += blockDim.x) {
        const unsigned long long h = mix((static_cast<unsigned long long>(blockIdx.x) << 32) ^ k);
        long long x;
        if (k & 1) {
            x = static_cast<long long>(h & ((1ull << 40) - 1));  // uniform in [0, 2^40)
        } else {  // a multiple of d, nudged by -2..+2
            const long long m = static_cast<long long>((h >> 8) & ((1ull << 40) - 1)) / d;
            x = m * d + static_cast<long long>(h & 3) - 2;
            if (x < 0) x = 0;
        }
        int r;
        const long long q = lsg::divmod_index(x, d, inv, r);
        ++cnt;
        if (q != x / d || r != static_cast<int>(x % d)) {
            ++bad;
            g_x = x;
            g_d = d;
        }
    }
    atomicAdd(&g_bad, bad);
    atomicAdd(&g_count, cnt);
}

int main() {
    check<<<65536 * 2, 256>>>(65536, 768);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) {
        std::printf("cuda error %s\n", cudaGetErrorString(e));
        return 2;
    }
    unsigned long long bad = 0, cnt = 0;
    long long x = 0;
    int d = 0;
    cudaMemcpyFromSymbol(&bad, g_bad, sizeof bad);
    cudaMemcpyFromSymbol(&cnt, g_count, sizeof cnt);
    cudaMemcpyFromSymbol(&x, g_x, sizeof x);
    cudaMemcpyFromSymbol(&d, g_d, sizeof d);
    if (bad) {
        std::printf("divmod MISMATCH %llu of %llu, e.g. x=%lld d=%d\n", bad, cnt, x, d);
        return 1;
    }
    std::printf("divmod ok %llu\n", cnt);
    return 0;
}
