// PCIe duplex probe: 1 GiB pinned H2D alone, D2H alone, and both at once on
// two streams (whole buffer, then in 32 MiB chunks) — the floor of the
// end-to-end step (lsg_solver_step_host copies the field in and out).
#include <cstdio>
#include <cuda_runtime.h>

int main() {
    const size_t n = 1ull << 30, chunk = 32ull << 20;
    void *h1, *h2, *d1, *d2;
    cudaMallocHost(&h1, n);
    cudaMallocHost(&h2, n);
    cudaMalloc(&d1, n);
    cudaMalloc(&d2, n);
    cudaStream_t a, b, a2, b2;
    cudaStreamCreateWithFlags(&a, cudaStreamNonBlocking);
    cudaStreamCreateWithFlags(&b, cudaStreamNonBlocking);
    cudaStreamCreateWithFlags(&a2, cudaStreamNonBlocking);
    cudaStreamCreateWithFlags(&b2, cudaStreamNonBlocking);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    auto run = [&](const char* name, int mode, size_t c) {
        float best = 1e30f;
        for (int rep = 0; rep < 3; ++rep) {
            cudaDeviceSynchronize();
            cudaEventRecord(e0, 0);
            for (cudaStream_t st : {a, b, a2, b2}) cudaStreamWaitEvent(st, e0, 0);
            const bool two = mode & 4;  // alternate chunks over two streams per direction
            size_t k = 0;
            for (size_t o = 0; o < n; o += c, ++k) {
                cudaStream_t sa = two && (k & 1) ? a2 : a, sb = two && (k & 1) ? b2 : b;
                if (mode & 1) cudaMemcpyAsync((char*)d1 + o, (char*)h1 + o, c, cudaMemcpyHostToDevice, sa);
                if (mode & 2) cudaMemcpyAsync((char*)h2 + o, (char*)d2 + o, c, cudaMemcpyDeviceToHost, sb);
            }
            for (cudaStream_t st : {a, b, a2, b2}) {
                cudaEvent_t ev;
                cudaEventCreate(&ev);
                cudaEventRecord(ev, st);
                cudaStreamWaitEvent(0, ev, 0);
            }
            cudaEventRecord(e1, 0);
            cudaEventSynchronize(e1);
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            if (ms < best) best = ms;
        }
        const double gb = (double)n * ((mode & 1) + ((mode >> 1) & 1)) / 1e9;
        printf("%-28s %8.2f ms  %6.1f GB/s total\n", name, best, gb / (best * 1e-3));
    };
    run("H2D 1 GiB", 1, n);
    run("D2H 1 GiB", 2, n);
    run("H2D + D2H concurrent", 3, n);
    run("H2D + D2H, 32 MiB chunks", 3, chunk);
    run("H2D, 2 streams, 32 MiB", 5, chunk);
    run("D2H, 2 streams, 32 MiB", 6, chunk);
    run("H2D + D2H, 2+2 streams", 7, chunk);
    run("H2D 32 MiB chunks", 1, chunk);
    return 0;
}
