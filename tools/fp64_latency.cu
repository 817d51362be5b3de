// tools/fp64_latency.cu — dependent-chain latency of DADD/DMUL/DSETP+FSEL and
// shared-memory loads on one warp (cycles per op, clock64).
#include <cstdio>
#include <cuda_runtime.h>

__global__ void lat(double* out, long long* cyc, int iters, double a) {
    __shared__ double sm[64];
    sm[threadIdx.x] = threadIdx.x;
    __syncthreads();
    double r = threadIdx.x * 1e-3;
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) r = __dadd_rn(r, a);
    long long t1 = clock64();
    for (int i = 0; i < iters; ++i) r = __dmul_rn(r, a);
    long long t2 = clock64();
    for (int i = 0; i < iters; ++i) r = fabs(r) <= fabs(a) ? r : a + r;  // DSETP + select + DADD
    long long t3 = clock64();
    int k = threadIdx.x;
    double acc = 0;
    for (int i = 0; i < iters; ++i) {
        acc = sm[(k + (int)acc) & 31];
    }
    long long t4 = clock64();
    out[threadIdx.x] = r + acc;
    if (threadIdx.x == 0) {
        cyc[0] = t1 - t0;
        cyc[1] = t2 - t1;
        cyc[2] = t3 - t2;
        cyc[3] = t4 - t3;
    }
}

int main() {
    double* out;
    long long* cyc;
    cudaMalloc(&out, 64 * sizeof(double));
    cudaMallocManaged(&cyc, 4 * sizeof(long long));
    const int iters = 4096;
    lat<<<1, 32>>>(out, cyc, iters, 1.0000001);
    lat<<<1, 32>>>(out, cyc, iters, 1.0000001);
    cudaDeviceSynchronize();
    printf("DADD chain %.2f cyc/op, DMUL chain %.2f, DSETP+sel+DADD %.2f, LDS.64 chain %.2f\n",
           (double)cyc[0] / iters, (double)cyc[1] / iters, (double)cyc[2] / iters, (double)cyc[3] / iters);
    return 0;
}
