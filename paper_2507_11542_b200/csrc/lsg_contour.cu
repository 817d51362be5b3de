// lsg_contour.cu — zero-set extraction of a 2-D field (contour.cpp:27-97) and
// 2-D slicing of a 3-D field (contour.cpp:99-135) on the device.
//
// Marching squares in three passes: per-cell segment counts (0, 1 or 2), an
// exclusive scan over cells in the reference's loop order (j outer, i inner),
// and segment emission at the scanned offsets — so the output order and every
// endpoint (IEEE division in the edge interpolation, no FMA) equal the
// reference's.
#include <cub/device/device_scan.cuh>

#include "lsg_misc.cuh"

namespace lsg {

namespace {

struct Pair {
    int a, b;
};

// Edge pairs per marching-squares code (contour.cpp:56-86); saddles 5 and 10
// split by the sign of the cell-centre average.
__device__ __forceinline__ int cell_pairs(double c0, double c1, double c2, double c3, Pair* p) {
    int code = 0;
    if (c0 < 0.0) code |= 1;
    if (c1 < 0.0) code |= 2;
    if (c2 < 0.0) code |= 4;
    if (c3 < 0.0) code |= 8;
    switch (code) {
        case 1: p[0] = {3, 0}; return 1;
        case 2: p[0] = {0, 1}; return 1;
        case 3: p[0] = {3, 1}; return 1;
        case 4: p[0] = {1, 2}; return 1;
        case 6: p[0] = {0, 2}; return 1;
        case 7: p[0] = {3, 2}; return 1;
        case 8: p[0] = {3, 2}; return 1;
        case 9: p[0] = {0, 2}; return 1;
        case 11: p[0] = {1, 2}; return 1;
        case 12: p[0] = {3, 1}; return 1;
        case 13: p[0] = {0, 1}; return 1;
        case 14: p[0] = {3, 0}; return 1;
        case 5: {
            const bool inside = 0.25 * (c0 + c1 + c2 + c3) < 0.0;
            if (inside) p[0] = {3, 2}, p[1] = {0, 1};
            else p[0] = {3, 0}, p[1] = {1, 2};
            return 2;
        }
        case 10: {
            const bool inside = 0.25 * (c0 + c1 + c2 + c3) < 0.0;
            if (inside) p[0] = {3, 0}, p[1] = {1, 2};
            else p[0] = {0, 1}, p[1] = {3, 2};
            return 2;
        }
    }
    return 0;
}

__device__ __forceinline__ double2 crossing(int edge, double x0, double y0, double dx, double dy, double c0, double c1,
                                            double c2, double c3) {
    // contour.cpp:14-23: lerp(va, vb) = va / (va - vb)
    switch (edge) {
        case 0: return make_double2(x0 + (c0 / (c0 - c1)) * dx, y0);
        case 1: return make_double2(x0 + dx, y0 + (c1 / (c1 - c2)) * dy);
        case 2: return make_double2(x0 + (c3 / (c3 - c2)) * dx, y0 + dy);
        default: return make_double2(x0, y0 + (c0 / (c0 - c3)) * dy);
    }
}

__global__ void count_kernel(const double* __restrict__ f, int nx, int ny, int* __restrict__ counts) {
    const int c = blockIdx.x * blockDim.x + threadIdx.x;
    const int ncx = nx - 1;
    if (c >= ncx * (ny - 1)) return;
    const int j = c / ncx, i = c - j * ncx;
    const long long b = (long long)j * nx + i;
    Pair p[2];
    counts[c] = cell_pairs(f[b], f[b + 1], f[b + 1 + nx], f[b + nx], p);
}

__global__ void emit_kernel(const double* __restrict__ f, int nx, int ny, const double* __restrict__ ax,
                            const double* __restrict__ ay, double dx, double dy, const int* __restrict__ offsets,
                            double* __restrict__ seg) {
    const int c = blockIdx.x * blockDim.x + threadIdx.x;
    const int ncx = nx - 1;
    if (c >= ncx * (ny - 1)) return;
    const int j = c / ncx, i = c - j * ncx;
    const long long b = (long long)j * nx + i;
    const double c0 = f[b], c1 = f[b + 1], c2 = f[b + 1 + nx], c3 = f[b + nx];
    Pair p[2];
    const int n = cell_pairs(c0, c1, c2, c3, p);
    for (int k = 0; k < n; ++k) {
        const double2 a = crossing(p[k].a, ax[i], ay[j], dx, dy, c0, c1, c2, c3);
        const double2 e = crossing(p[k].b, ax[i], ay[j], dx, dy, c0, c1, c2, c3);
        double* o = seg + 4LL * (offsets[c] + k);
        o[0] = a.x, o[1] = a.y, o[2] = e.x, o[3] = e.y;
    }
}

__global__ void slice_kernel(const double* __restrict__ f, long long total, int n0, long long s0, long long s1,
                             long long fixed_offset, double* __restrict__ out) {
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= total) return;
    const long long a = i % n0, b = i / n0;
    out[i] = f[fixed_offset + a * s0 + b * s1];
}

}  // namespace

// Count, scan and emit; returns the number of segments (written when it fits).
long long zero_set_2d(const double* f, int nx, int ny, const double* ax, const double* ay, double dx, double dy,
                      double* seg_dev, long long cap, int* scratch_counts, int* scratch_offsets, void* temp,
                      size_t temp_bytes, cudaStream_t st, int* total_host) {
    const int ncells = (nx - 1) * (ny - 1);
    const unsigned blocks = (unsigned)((ncells + 255) / 256);
    count_kernel<<<blocks, 256, 0, st>>>(f, nx, ny, scratch_counts);
    size_t tb = temp_bytes;
    cub::DeviceScan::ExclusiveSum(temp, tb, scratch_counts, scratch_offsets, ncells, st);
    int last_off = 0, last_cnt = 0;
    cudaMemcpyAsync(&last_off, scratch_offsets + ncells - 1, sizeof(int), cudaMemcpyDeviceToHost, st);
    cudaMemcpyAsync(&last_cnt, scratch_counts + ncells - 1, sizeof(int), cudaMemcpyDeviceToHost, st);
    cudaStreamSynchronize(st);
    *total_host = last_off + last_cnt;
    if (*total_host <= cap && *total_host > 0)
        emit_kernel<<<blocks, 256, 0, st>>>(f, nx, ny, ax, ay, dx, dy, scratch_offsets, seg_dev);
    return *total_host;
}

size_t zero_set_temp_bytes(int ncells) {
    size_t tb = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, tb, (int*)nullptr, (int*)nullptr, ncells);
    return tb;
}

void launch_slice(const double* f, long long total, int n0, long long s0, long long s1, long long fixed_offset,
                  double* out, cudaStream_t st) {
    slice_kernel<<<(unsigned)((total + 255) / 256), 256, 0, st>>>(f, total, n0, s0, s1, fixed_offset, out);
}

}  // namespace lsg
