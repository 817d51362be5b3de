// Bitwise check of the exact WENO5 building blocks (lsg_device.cuh) against
// the reference's arithmetic with plain IEEE division (weno5_onesided,
// spatial_derivatives.cpp:78-97, as weno5_onesided_impl<true>):
//   * div_by3 / div_by6 (the select-free constant division) on random
//     doubles over the admitted exponent range, zeros of both signs, small
//     integers, and the range edges;
//   * line_lr<WENO5> (one node) and line_lr2<WENO5> (two adjacent nodes with
//     shared quotients) on random windows: first differences of mixed
//     magnitudes, exact zeros, repeated values, subnormal-adjacent and
//     huge differences (which take the out-of-line IEEE path).
// Prints "weno5 ok <n>" or the first mismatch; built by __graft_entry__.build(),
// run by tests/test_gpu_shim.py.
#include <cstdio>
#include <cuda_runtime.h>

#include "../../paper_2507_11542_b200/csrc/lsg_device.cuh"

using namespace lsg;

__device__ unsigned long long g_bad = 0, g_count = 0;
__device__ int g_kind = 0;
__device__ double g_x = 0.0;

__device__ __forceinline__ unsigned long long mix(unsigned long long z) {
    z += 0x9e3779b97f4a7c15ull;
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
    return z ^ (z >> 31);
}

__device__ bool same(double a, double b) {
    return __double_as_longlong(a) == __double_as_longlong(b) || (a != a && b != b);
}

__device__ void report(int kind, double x) {
    if (atomicAdd(&g_bad, 1ull) == 0) {
        g_kind = kind;
        g_x = x;
    }
}

// division: x over the exponent range div_const admits, plus edge values
__global__ void check_div(unsigned long long seed, long long n) {
    unsigned long long cnt = 0;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
        unsigned long long b = mix(seed + i);
        const unsigned long long be = 66 + (b >> 52) % (2023 - 66);  // 2^-957 <= |x| < 2^1000
        b = (b & 0x800FFFFFFFFFFFFFull) | (be << 52);
        double x = __longlong_as_double((long long)b);
        if ((i & 1023) == 0) x = (double)((long long)(b % 2001) - 1000);
        if (i == 0) x = -0.0;
        if (i == 1) x = 0.0;
        if (i == 2) x = 0x1p-957;
        if (i == 3) x = -0x1p-957;
        if (i == 4) x = __longlong_as_double(0x7E6FFFFFFFFFFFFFll);  // largest admitted
        if (i == 5) x = 3.0;
        if (i == 6) x = -6.0;
        if (i == 7) x = 0x1p-250;
        if (i == 8) x = -0x1.fffffffffffffp+249;  // largest the fast path admits
        if (i == 9) x = 0x1p250;                  // smallest it refuses above
        if (i == 10) x = 0x1.fffffffffffffp-251;  // largest it refuses below
        // the fast path's operand test admits exactly +-0 and 2^-250 <= |x| < 2^250
        // (a subset of the range checked for the divisions here)
        const double ax = fabs(x);
        if (weno5_operand_ok(x) != (ax == 0.0 || (ax >= 0x1p-250 && ax < 0x1p250))) report(1, x);
        if (!same(div_by3(x), x / 3.0) || !same(div_by6(x), x / 6.0)) report(2, x);
        if (!same(0.5 * div_by3(x), x / 6.0)) report(3, x);
        ++cnt;
    }
    atomicAdd(&g_count, cnt);
}

__device__ double draw(unsigned long long h, int mode) {
    // a window value: smooth-ish, with the distributions that stress the domains
    const double u = (double)(h >> 11) * 0x1p-53;  // [0, 1)
    switch (mode) {
        case 0: return u * 2.0 - 1.0;                                           // O(1)
        case 1: return (double)((long long)(h % 7) - 3);                         // small integers: exact zeros, ties
        case 2: return ldexp(u * 2.0 - 1.0, (int)((h >> 3) % 200) - 100);      // mixed magnitudes
        case 3: return ldexp(u, -1000 - (int)(h % 60));                          // subnormal-adjacent differences
        case 4: return ldexp(u * 2.0 - 1.0, 900 + (int)(h % 120));              // huge (and overflowing) values
        case 6: return ldexp(u * 2.0 - 1.0, ((h >> 7) & 1 ? -262 : 238) + (int)((h >> 3) % 16));  // edges of the fast path's range
        default: return (h & 1) ? 0.0 : -0.0;                                    // signed zeros
    }
}

__global__ void check_lr(unsigned long long seed, long long n, LineConst c) {
    unsigned long long cnt = 0;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
        const unsigned long long h0 = mix(seed ^ (unsigned long long)i);
        const int mode = (int)(h0 % 16);
        double s[8];
        for (int j = 0; j < 8; ++j) {
            const unsigned long long h = mix(h0 + 0x51ull * (j + 1));
            s[j] = draw(h, mode < 5 ? 0 : mode < 8 ? 1 : mode < 11 ? 2 : mode < 12 ? 3 : mode < 13 ? 4 : mode < 14 ? 5 : mode < 15 ? 6 : (int)(h % 7));
            if (mode == 7 && j > 0 && (h & 3) == 0) s[j] = s[j - 1];  // flat runs
        }
        // reference: plain IEEE divisions in the reference's order
        double d1[7];
        for (int j = 0; j < 7; ++j) d1[j] = (s[j + 1] - s[j]) * c.inv_dx;
        bool unused;
        const double La = weno5_onesided_impl<true>(d1[0], d1[1], d1[2], d1[3], d1[4], unused);
        const double Ra = weno5_onesided_impl<true>(d1[5], d1[4], d1[3], d1[2], d1[1], unused);
        const double Lb = weno5_onesided_impl<true>(d1[1], d1[2], d1[3], d1[4], d1[5], unused);
        const double Rb = weno5_onesided_impl<true>(d1[6], d1[5], d1[4], d1[3], d1[2], unused);
        double L, R, L2, R2, L3, R3;
        line_lr<WENO5>(s, c, L, R);
        line_lr2<WENO5>(s, c, L2, R2, L3, R3);
        if (!same(L, La) || !same(R, Ra)) report(10 + mode, s[3]);
        if (!same(L2, La) || !same(R2, Ra) || !same(L3, Lb) || !same(R3, Rb)) report(30 + mode, s[3]);
        ++cnt;
    }
    atomicAdd(&g_count, cnt);
}

int main() {
    unsigned long long bad = 0, cnt = 0;
    const long long nd = 1LL << 30;
    check_div<<<148 * 8, 256>>>(0x1234567ull, nd);
    LineConst c{};
    for (int k = 0; k < 3; ++k) {
        const double dx = k == 0 ? 2.0 / 512.0 : k == 1 ? 0.05 : 1.0 / 3.0;
        c.dx = dx;
        c.inv_dx = 1.0 / dx;
        c.half_inv = 0.5 * c.inv_dx;
        c.third_inv = c.inv_dx / 3.0;
        c.dx2 = dx * dx;
        check_lr<<<148 * 8, 256>>>(0xabcdefull + 977 * k, 1LL << 26, c);
    }
    if (cudaDeviceSynchronize() != cudaSuccess) {
        printf("weno5 check: CUDA error %s\n", cudaGetErrorString(cudaGetLastError()));
        return 2;
    }
    cudaMemcpyFromSymbol(&bad, g_bad, sizeof bad);
    cudaMemcpyFromSymbol(&cnt, g_count, sizeof cnt);
    if (bad) {
        int kind = 0;
        double x = 0.0;
        cudaMemcpyFromSymbol(&kind, g_kind, sizeof kind);
        cudaMemcpyFromSymbol(&x, g_x, sizeof x);
        printf("weno5 MISMATCH: %llu of %llu; first kind %d at %a\n", bad, cnt, kind, x);
        return 1;
    }
    printf("weno5 ok %llu\n", cnt);
    return 0;
}
