// lsg_misc.cuh — host-visible launchers and lookup tables of the device kernels.
#pragma once

#include <cuda_runtime.h>

#include "lsg_box3.cuh"
#include "lsg_march3.cuh"
#include "lsg_marchn.cuh"

namespace lsg {

struct ShapeParams {
    long long n_local;
    int D;
    int n[kMaxDim];
    int z0;
    const double* axis[kMaxDim];
    int shape;             // 0 sphere, 1 cylinder, 2 planar pair distance, 3 rectangle, 4 ellipsoid
    int op;                // 0 replace, 1 union (std::min), 2 intersection (std::max) with out
    unsigned ignored_mask;
    double center[kMaxDim];  // sphere/cylinder centre; rectangle lower corner
    double upper[kMaxDim];   // rectangle upper corner
    double radius;
    double* out;
};

using AlphaFn = void (*)(AlphaParams);

Box3Fn box3_lookup_linear(int s, int m, bool range);
Box3Fn box3_lookup_normal(int s, int m, bool range);
Box3Fn box3_lookup_rockets(int s, int m, bool range);
Box3Fn box3_lookup_air3d(int s, int m, bool range);
March3Fn march3_lookup_linear(int s, int m, bool range);
March3Fn march3_lookup_normal(int s, int m, bool range);
March3Fn march3_lookup_rockets(int s, int m, bool range);
March3Fn march3_lookup_air3d(int s, int m, bool range);
March3TmaFn march3_tma_lookup_linear(int s, int m, bool range);
MarchNFn marchn_lookup_linear(int D, int s, int m, bool range);
MarchNFn marchn_lookup_dblint4(int D, int s, int m, bool range);
MarchNFn marchn_lookup_dubins6(int D, int s, int m, bool range);
March3TmaFn march3_tma_lookup_normal(int s, int m, bool range);
March3TmaFn march3_tma_lookup_rockets(int s, int m, bool range);
March3TmaFn march3_tma_lookup_air3d(int s, int m, bool range);

StageFn stage_lookup_linear(int D, int s, int m);
StageFn stage_lookup_normal(int D, int s, int m);
StageFn stage_lookup_rotation(int D, int s, int m);
StageFn stage_lookup_rockets(int D, int s, int m);
StageFn stage_lookup_air3d(int D, int s, int m);
StageFn stage_lookup_dblint4(int D, int s, int m);
StageFn stage_lookup_dubins6(int D, int s, int m);
EvalFn eval_lookup_linear(int D);
EvalFn eval_lookup_normal(int D);
EvalFn eval_lookup_rotation(int D);
EvalFn eval_lookup_rockets(int D);
EvalFn eval_lookup_air3d(int D);
EvalFn eval_lookup_dblint4(int D);
EvalFn eval_lookup_dubins6(int D);
AlphaFn alpha_lookup_linear();
AlphaFn alpha_lookup_normal();
AlphaFn alpha_lookup_rotation();
AlphaFn alpha_lookup_rockets();
AlphaFn alpha_lookup_air3d();
AlphaFn alpha_lookup_dblint4();
AlphaFn alpha_lookup_dubins6();

void launch_upwind(const StageParams& P, int dim, int D, int scheme, double* left, double* right, cudaStream_t st);
void launch_pad(const double* u, double* out, long long n_out, int n, long long stride, int width, int bc,
                cudaStream_t st);
void launch_shift(const double* padded, double* out, long long N, int n, long long stride, int width, int offset,
                  cudaStream_t st);
void launch_restrict(const double* in, double* out, long long n, int direction, cudaStream_t st);
void launch_shape(const ShapeParams& S, cudaStream_t st);
// elementwise set operations (implicit_surfaces.cpp:128-151): op 1 min, 2 max, 3 negate a
void launch_set_op(int op, long long n, const double* a, const double* b, double* out, cudaStream_t st);
void launch_stamp(unsigned long long* out, cudaStream_t st);  // %globaltimer into *out (tracing)
// blocks x 256 threads x 8 chains x iters FP64 DADD/DMUL (lsg_probe_fp64_rate)
void launch_fp64_rate(double* out, int blocks, int iters, cudaStream_t st);
void launch_range_init(unsigned long long* r, long long nslots, cudaStream_t st);
long long zero_set_2d(const double* f, int nx, int ny, const double* ax, const double* ay, double dx, double dy,
                      double* seg_dev, long long cap, int* scratch_counts, int* scratch_offsets, void* temp,
                      size_t temp_bytes, cudaStream_t st, int* total_host);
size_t zero_set_temp_bytes(int ncells);
void launch_slice(const double* f, long long total, int n0, long long s0, long long s1, long long fixed_offset,
                  double* out, cudaStream_t st);

}  // namespace lsg
