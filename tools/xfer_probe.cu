// Host<->device transfer paths for the reference-facing API (std::vector
// buffers): pageable cudaMemcpyAsync vs pinned vs a chunked copy staged
// through two pinned buffers with std::memcpy (1 and 4 threads).
#include <chrono>
#include <cstdio>
#include <cstring>
#include <thread>
#include <vector>
#include <cuda_runtime.h>

static double now() {
    return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

static void par_memcpy(void* d, const void* s, size_t n, int threads) {
    if (threads <= 1) { std::memcpy(d, s, n); return; }
    std::vector<std::thread> ts;
    size_t per = (n + threads - 1) / threads;
    for (int t = 0; t < threads; ++t) {
        size_t a = t * per, b = std::min(n, a + per);
        if (a >= b) break;
        ts.emplace_back([=] { std::memcpy((char*)d + a, (const char*)s + a, b - a); });
    }
    for (auto& t : ts) t.join();
}

int main() {
    cudaStream_t st;
    cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
    const size_t chunk = 4 << 20;
    char* pin[2];
    cudaMallocHost((void**)&pin[0], chunk);
    cudaMallocHost((void**)&pin[1], chunk);
    cudaEvent_t ev[2];
    cudaEventCreate(&ev[0]); cudaEventCreate(&ev[1]);
    for (size_t mb : {2, 8, 64}) {
        size_t n = mb << 20;
        std::vector<char> host(n, 1);
        char* ph; cudaMallocHost((void**)&ph, n);
        char* dv; cudaMalloc((void**)&dv, n);
        auto timeit = [&](auto f) { f(); cudaStreamSynchronize(st); double t = now(); for (int i = 0; i < 10; ++i) f(); cudaStreamSynchronize(st); return (now() - t) / 10; };
        double t_pg_h2d = timeit([&] { cudaMemcpyAsync(dv, host.data(), n, cudaMemcpyHostToDevice, st); cudaStreamSynchronize(st); });
        double t_pg_d2h = timeit([&] { cudaMemcpyAsync(host.data(), dv, n, cudaMemcpyDeviceToHost, st); cudaStreamSynchronize(st); });
        double t_pn_h2d = timeit([&] { cudaMemcpyAsync(dv, ph, n, cudaMemcpyHostToDevice, st); cudaStreamSynchronize(st); });
        double t_pn_d2h = timeit([&] { cudaMemcpyAsync(ph, dv, n, cudaMemcpyDeviceToHost, st); cudaStreamSynchronize(st); });
        for (int th : {1, 4}) {
            double t_st_h2d = timeit([&] {
                for (size_t off = 0, k = 0; off < n; off += chunk, ++k) {
                    size_t b = std::min(chunk, n - off);
                    cudaEventSynchronize(ev[k & 1]);
                    par_memcpy(pin[k & 1], host.data() + off, b, th);
                    cudaMemcpyAsync(dv + off, pin[k & 1], b, cudaMemcpyHostToDevice, st);
                    cudaEventRecord(ev[k & 1], st);
                }
                cudaStreamSynchronize(st);
            });
            double t_st_d2h = timeit([&] {
                size_t nchunks = (n + chunk - 1) / chunk;
                for (size_t k = 0; k < nchunks + 1; ++k) {
                    if (k < nchunks) {
                        size_t off = k * chunk, b = std::min(chunk, n - off);
                        cudaEventSynchronize(ev[k & 1]);  // buffer free (drained below)
                        cudaMemcpyAsync(pin[k & 1], dv + off, b, cudaMemcpyDeviceToHost, st);
                        cudaEventRecord(ev[k & 1], st);
                    }
                    if (k >= 1) {
                        size_t j = k - 1, off = j * chunk, b = std::min(chunk, n - off);
                        cudaEventSynchronize(ev[j & 1]);
                        par_memcpy(host.data() + off, pin[j & 1], b, th);
                    }
                }
            });
            printf("%3zu MB staged(%d thr): h2d %.2f GB/s d2h %.2f GB/s\n", mb, th, n / t_st_h2d / 1e9, n / t_st_d2h / 1e9);
        }
        printf("%3zu MB pageable: h2d %.2f GB/s d2h %.2f GB/s | pinned: h2d %.2f d2h %.2f GB/s\n", mb,
               n / t_pg_h2d / 1e9, n / t_pg_d2h / 1e9, n / t_pn_h2d / 1e9, n / t_pn_d2h / 1e9);
        cudaFreeHost(ph); cudaFree(dv);
    }
    return 0;
}
