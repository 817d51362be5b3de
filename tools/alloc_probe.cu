// cudaMalloc/cudaFree vs the stream-ordered pool (cudaMallocAsync with a
// retained pool) for the solver's buffer set at 101^3 (3 x 8.2 MB + tables).
#include <chrono>
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

static double now() {
    return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

int main() {
    const size_t field = 101ull * 101 * 101 * 8;
    const size_t sizes[] = {field, field, field, 4096, 65536, 8, 64};
    cudaFree(0);
    cudaStream_t st;
    cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
    for (int rep = 0; rep < 2; ++rep) {
        double t0 = now();
        for (int it = 0; it < 20; ++it) {
            void* p[7];
            for (int k = 0; k < 7; ++k) cudaMalloc(&p[k], sizes[k]);
            for (int k = 0; k < 7; ++k) cudaFree(p[k]);
        }
        double t1 = now();
        printf("cudaMalloc+cudaFree set: %.3f ms\n", (t1 - t0) / 20);
    }
    cudaMemPool_t pool;
    cudaDeviceGetDefaultMemPool(&pool, 0);
    uint64_t thr = UINT64_MAX;
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
    for (int rep = 0; rep < 2; ++rep) {
        double t0 = now();
        for (int it = 0; it < 20; ++it) {
            void* p[7];
            for (int k = 0; k < 7; ++k) cudaMallocAsync(&p[k], sizes[k], st);
            for (int k = 0; k < 7; ++k) cudaFreeAsync(p[k], st);
            cudaStreamSynchronize(st);
        }
        double t1 = now();
        printf("pool set: %.3f ms\n", (t1 - t0) / 20);
    }
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
