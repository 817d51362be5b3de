// tools/fp64_peak.cu — measures the FP64 (DADD/DMUL, no FMA) issue rate of one
// B200, the second roofline of the HJ stencil.  Each thread runs
// 8 independent dependency chains; grid = 148 * 8 blocks of 256 threads.
#include <cstdio>
#include <cuda_runtime.h>

template <int OP>
__global__ void chains(double* out, int iters, double a, double b) {
    double r[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) r[k] = threadIdx.x * 1e-3 + k;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            if (OP == 0) r[k] = __dadd_rn(r[k], a);
            else if (OP == 1) r[k] = __dmul_rn(r[k], b);
            else r[k] = __dadd_rn(__dmul_rn(r[k], b), a);
        }
    }
    double s = 0;
#pragma unroll
    for (int k = 0; k < 8; ++k) s += r[k];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const int blocks = sms * 8, threads = 256, iters = 20000;
    double* out;
    cudaMalloc(&out, sizeof(double) * blocks * threads);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const char* names[3] = {"DADD", "DMUL", "DMUL+DADD"};
    for (int op = 0; op < 3; ++op) {
        for (int rep = 0; rep < 2; ++rep) {
            cudaEventRecord(e0);
            if (op == 0) chains<0><<<blocks, threads>>>(out, iters, 1e-9, 1.0000001);
            if (op == 1) chains<1><<<blocks, threads>>>(out, iters, 1e-9, 1.0000001);
            if (op == 2) chains<2><<<blocks, threads>>>(out, iters, 1e-9, 1.0000001);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            const double ops = double(blocks) * threads * iters * 8 * (op == 2 ? 2 : 1);
            if (rep) printf("%-10s %.3f ms  %.2f T FP64 instr/s  = %.1f per SM per ns\n", names[op], ms,
                            ops / ms * 1e-9, ops / ms * 1e-6 / sms);
        }
    }
    int clk = 0;
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    printf("SMs %d, max clock %d MHz\n", sms, clk / 1000);
    return 0;
}
