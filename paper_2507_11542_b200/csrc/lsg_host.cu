// lsg_host.cu — host runtime and C ABI of the B200 HJ hot path (include/lsg.h).
//
// Owns contexts (device + stream [+ NCCL communicator]), device-resident
// solvers (value function slabs in HBM, coordinate/trig tables, the global
// Lax-Friedrichs alpha), the exact step control of the reference integrator
// and the slab halo exchange.
//
// Step control.  The reference's dissipation bound takes (t, grid, dim) and
// never the value function (hamiltonian.hpp:24-25), and every device kind is
// time-invariant, so alpha, the CFL bound and therefore the whole dt sequence
// of a leg are known before any stage runs.  run_cfl below replays the
// reference loop (integrator.cpp:22-97) on the host to build that schedule,
// enqueues every stage of the leg back to back with no host synchronisation,
// and synchronises once at the end of the leg to collect the per-step v range
// (fused into the last stage of each step) and the error flags.
//
// Also here: the stream-ordered device pool and the per-context solver cache
// of the stateless calls; slabs (halo planes, boundary bands on a side
// stream, the halo exchange on a communication stream overlapped with the
// interior, NCCL for ranks / device copies in process); and
// lsg_solver_step_host (host-to-host step, copies chunked along the slab axis
// and overlapped with the stage kernels).
#include <cuda_runtime.h>
#include <nccl.h>
#include <nvtx3/nvToolsExt.h>  // header-only; ranges cost nothing unless a tool is attached

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <fstream>
#include <sstream>
#include <cstdlib>
#include <cstring>
#include <limits>
#include <memory>
#include <mutex>
#include <new>
#include <string>
#include <vector>

#include "lsg_misc.cuh"

using namespace lsg;

namespace {

thread_local std::string g_err;

struct Error {
    int code;
    std::string msg;
};

[[noreturn]] void fail(int code, const std::string& msg) { throw Error{code, msg}; }

#define CUDA_CHECK(x)                                                                         \
    do {                                                                                      \
        cudaError_t e_ = (x);                                                                 \
        if (e_ != cudaSuccess) fail(LSG_ECUDA, std::string(#x) + ": " + cudaGetErrorString(e_)); \
    } while (0)

#define NCCL_CHECK(x)                                                                           \
    do {                                                                                        \
        ncclResult_t r_ = (x);                                                                  \
        if (r_ != ncclSuccess) fail(LSG_ENCCL, std::string(#x) + ": " + ncclGetErrorString(r_)); \
    } while (0)

template <typename F>
int guarded(F&& f) {
    try {
        f();
        return LSG_OK;
    } catch (const Error& e) {
        g_err = e.msg;
        return e.code;
    } catch (const std::bad_alloc&) {
        g_err = "host allocation failed";
        return LSG_ENOMEM;
    } catch (const std::exception& e) {
        g_err = e.what();
        return LSG_EINVAL;
    }
}

// Device buffers come from a per-device stream-ordered pool owned by the
// library: building and tearing down a solver then costs microseconds instead
// of the milliseconds cudaMalloc/cudaFree take (tools/alloc_probe.cu).  The
// pool keeps up to kPoolKeep bytes of freed memory for reuse and returns the
// rest to the device at the next synchronisation, so it does not hoard memory
// from other allocators in the process (e.g. torch's).
constexpr uint64_t kPoolKeep = 1ull << 30;

cudaMemPool_t lib_pool(int device) {
    static std::mutex m;
    static cudaMemPool_t pools[256] = {};
    std::lock_guard<std::mutex> lock(m);
    if (device < 0 || device >= 256) fail(LSG_EINVAL, "device ordinal out of range");
    if (!pools[device]) {
        cudaMemPoolProps props{};
        props.allocType = cudaMemAllocationTypePinned;
        props.location.type = cudaMemLocationTypeDevice;
        props.location.id = device;
        cudaMemPool_t pool = nullptr;
        cudaError_t e = cudaMemPoolCreate(&pool, &props);
        if (e != cudaSuccess) {
            cudaGetLastError();
            fail(LSG_ECUDA, std::string("cudaMemPoolCreate: ") + cudaGetErrorString(e));
        }
        uint64_t keep = kPoolKeep;
        cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
        pools[device] = pool;
    }
    return pools[device];
}

struct DevBuf {
    void* p = nullptr;
    size_t bytes = 0;
    cudaStream_t st = nullptr;  // allocation / release stream (the owning context's)
    DevBuf() = default;
    DevBuf(const DevBuf&) = delete;
    DevBuf& operator=(const DevBuf&) = delete;
    DevBuf(DevBuf&& o) noexcept : p(o.p), bytes(o.bytes), st(o.st) { o.p = nullptr, o.bytes = 0; }
    ~DevBuf() { release(); }
    void release() {
        if (p) cudaFreeAsync(p, st);
        p = nullptr;
        bytes = 0;
    }
    // Stream-ordered on `stream`; callers synchronise it before handing the
    // memory to other streams (make_solver does, staging users stay on it).
    void alloc(size_t b, cudaStream_t stream) {
        release();
        st = stream;
        if (b == 0) return;
        int dev = 0;
        cudaGetDevice(&dev);
        cudaMemPool_t pool = lib_pool(dev);
        cudaError_t e = cudaMallocFromPoolAsync(&p, b, pool, stream);
        if (e == cudaErrorMemoryAllocation) {  // hand retained memory back and retry once
            cudaGetLastError();
            cudaStreamSynchronize(stream);
            cudaMemPoolTrimTo(pool, 0);
            e = cudaMallocFromPoolAsync(&p, b, pool, stream);
        }
        if (e != cudaSuccess) {
            p = nullptr;
            cudaGetLastError();
            fail(LSG_ENOMEM, "device allocation of " + std::to_string(b) + " bytes failed: " + cudaGetErrorString(e));
        }
        bytes = b;
    }
    template <typename T>
    T* as() const {
        return static_cast<T*>(p);
    }
};

// ---- grid helpers (grid.cpp:9-66) ------------------------------------------

void check_grid(const lsg_grid* g) {
    if (!g) fail(LSG_EINVAL, "grid: null descriptor");
    if (g->dim <= 0) fail(LSG_EINVAL, "grid: dimension must be at least 1");
    if (g->dim > LSG_MAX_DIM) fail(LSG_EINVAL, "grid: at most 6 dimensions are supported");
    for (int d = 0; d < g->dim; ++d) {
        if (g->counts[d] < 3) fail(LSG_EINVAL, "grid: counts[" + std::to_string(d) + "] must be >= 3");
        if (!(g->maxs[d] > g->mins[d]))
            fail(LSG_EINVAL, "grid: max must exceed min in dimension " + std::to_string(d));
    }
    if (g->periodic_mask >> g->dim) fail(LSG_EINVAL, "grid: periodic dimension out of range");
}

double spacing(const lsg_grid* g, int d) {  // grid.cpp:41
    return (g->maxs[d] - g->mins[d]) / static_cast<double>(g->counts[d] - 1);
}

long long node_count(const lsg_grid* g) {
    long long n = 1;
    for (int d = 0; d < g->dim; ++d) n *= g->counts[d];
    return n;
}

int bc_of(const lsg_grid* g, int d) { return (g->periodic_mask >> d) & 1u ? LSG_BC_PERIODIC : LSG_BC_EXTRAPOLATE; }

int ghost_width(int scheme) {  // spatial_derivatives.cpp:10-18
    switch (scheme) {
        case LSG_SCHEME_FIRST: return 1;
        case LSG_SCHEME_ENO2: return 2;
        case LSG_SCHEME_ENO3: return 3;
        case LSG_SCHEME_WENO5: return 3;
    }
    fail(LSG_EINVAL, "unknown derivative scheme");
}

int min_nodes(int scheme) {  // spatial_derivatives.cpp:20-28
    switch (scheme) {
        case LSG_SCHEME_FIRST: return 3;
        case LSG_SCHEME_ENO2: return 5;
        case LSG_SCHEME_ENO3: return 7;
        case LSG_SCHEME_WENO5: return 7;
    }
    fail(LSG_EINVAL, "unknown derivative scheme");
}

const char* scheme_name(int scheme) {
    switch (scheme) {
        case LSG_SCHEME_FIRST: return "upwind_first_first";
        case LSG_SCHEME_ENO2: return "upwind_first_eno2";
        case LSG_SCHEME_ENO3: return "upwind_first_eno3";
        default: return "upwind_first_weno5";
    }
}

LineConst line_const(const lsg_grid* g, int d) {
    LineConst c;
    c.dx = spacing(g, d);
    c.inv_dx = 1.0 / c.dx;
    c.half_inv = 0.5 * c.inv_dx;
    c.third_inv = c.inv_dx / 3.0;
    c.dx2 = c.dx * c.dx;
    c.hs6 = 0.5 * (c.inv_dx * (1.0 / 6.0));
    return c;
}

}  // namespace

// ---- context -----------------------------------------------------------------

struct lsg_ctx {
    int device = 0;
    cudaStream_t stream = nullptr;
    uint64_t launches = 0;
    int rank = 0;
    int nranks = 1;
    bool dist_selftest = false;  // one-rank communicator driving the distributed branch (LSG_DIST_SELFTEST)
    ncclComm_t comm = nullptr;
    DevBuf scratch[4];  // stateless-call staging
    lsg_solver* cached = nullptr;  // last solver built by a stateless call (see cached_solver)
    std::string cached_key;

    void note_launch(int n = 1) {
        launches += static_cast<uint64_t>(n);
        const cudaError_t e = cudaGetLastError();
        if (e != cudaSuccess) fail(LSG_ECUDA, std::string("kernel launch: ") + cudaGetErrorString(e));
    }
    double* staging(int k, size_t bytes) {
        if (scratch[k].bytes < bytes) scratch[k].alloc(bytes, stream);
        return scratch[k].as<double>();
    }
};

namespace {

// NVTX range around host-side enqueue work (tracing): the names
// tie a profiler timeline's launches to the reference's loop structure
// (integrator.cpp:58-85 stages, reachability.cpp:160-170 legs).
struct NvtxRange {
    bool on;
    NvtxRange(bool enabled, const char* name) : on(enabled) {
        if (on) nvtxRangePushA(name);
    }
    ~NvtxRange() {
        if (on) nvtxRangePop();
    }
};

void activate(lsg_ctx* ctx) {
    if (!ctx) fail(LSG_EINVAL, "null context");
    CUDA_CHECK(cudaSetDevice(ctx->device));
}

StageFn lookup_stage(int kind, int D, int scheme, int mode) {
    switch (kind) {
        case LSG_HAM_LINEAR: return stage_lookup_linear(D, scheme, mode);
        case LSG_HAM_NORMAL: return stage_lookup_normal(D, scheme, mode);
        case LSG_HAM_ROTATION: return stage_lookup_rotation(D, scheme, mode);
        case LSG_HAM_ROCKETS: return stage_lookup_rockets(D, scheme, mode);
        case LSG_HAM_AIR3D: return stage_lookup_air3d(D, scheme, mode);
        case LSG_HAM_DBLINT4: return stage_lookup_dblint4(D, scheme, mode);
        case LSG_HAM_DUBINS6: return stage_lookup_dubins6(D, scheme, mode);
    }
    return nullptr;
}

March3Fn lookup_march3(int kind, int scheme, int mode, bool range) {
    switch (kind) {
        case LSG_HAM_LINEAR: return march3_lookup_linear(scheme, mode, range);
        case LSG_HAM_NORMAL: return march3_lookup_normal(scheme, mode, range);
        case LSG_HAM_ROCKETS: return march3_lookup_rockets(scheme, mode, range);
        case LSG_HAM_AIR3D: return march3_lookup_air3d(scheme, mode, range);
    }
    return nullptr;
}

MarchNFn lookup_marchn(int kind, int D, int scheme, int mode, bool range) {
    switch (kind) {
        case LSG_HAM_LINEAR: return marchn_lookup_linear(D, scheme, mode, range);
        case LSG_HAM_DBLINT4: return marchn_lookup_dblint4(D, scheme, mode, range);
        case LSG_HAM_DUBINS6: return marchn_lookup_dubins6(D, scheme, mode, range);
    }
    return nullptr;
}

March3TmaFn lookup_march3_tma(int kind, int scheme, int mode, bool range) {
    switch (kind) {
        case LSG_HAM_LINEAR: return march3_tma_lookup_linear(scheme, mode, range);
        case LSG_HAM_NORMAL: return march3_tma_lookup_normal(scheme, mode, range);
        case LSG_HAM_ROCKETS: return march3_tma_lookup_rockets(scheme, mode, range);
        case LSG_HAM_AIR3D: return march3_tma_lookup_air3d(scheme, mode, range);
    }
    return nullptr;
}

// cuTensorMapEncodeTiled through the runtime's driver entry point (no -lcuda).
using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                   const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                   CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
EncodeTiledFn encode_tiled() {
    static EncodeTiledFn fn = [] {
        void* f = nullptr;
        cudaDriverEntryPointQueryResult q{};
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess) {
            cudaGetLastError();
            return static_cast<EncodeTiledFn>(nullptr);
        }
        return reinterpret_cast<EncodeTiledFn>(f);
    }();
    return fn;
}

// 3-D fp64 tensor map over a slab buffer of n0 x n1 x nz doubles (plane -halo
// first), box bx x by x 1, zero fill outside.
CUtensorMap tensor_map_3d(const double* base, int n0, int n1, int nz, int bx, int by) {
    CUtensorMap m;
    const cuuint64_t dims[3] = {static_cast<cuuint64_t>(n0), static_cast<cuuint64_t>(n1), static_cast<cuuint64_t>(nz)};
    const cuuint64_t strides[2] = {sizeof(double) * static_cast<cuuint64_t>(n0),
                                   sizeof(double) * static_cast<cuuint64_t>(n0) * static_cast<cuuint64_t>(n1)};
    const cuuint32_t box[3] = {static_cast<cuuint32_t>(bx), static_cast<cuuint32_t>(by), 1u};
    const cuuint32_t estr[3] = {1u, 1u, 1u};
    const CUresult r = encode_tiled()(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, const_cast<double*>(base), dims, strides,
                                      box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                      CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) fail(LSG_ECUDA, "cuTensorMapEncodeTiled failed (" + std::to_string(static_cast<int>(r)) + ")");
    return m;
}

Box3Fn lookup_box3(int kind, int scheme, int mode, bool range) {
    switch (kind) {
        case LSG_HAM_LINEAR: return box3_lookup_linear(scheme, mode, range);
        case LSG_HAM_NORMAL: return box3_lookup_normal(scheme, mode, range);
        case LSG_HAM_ROCKETS: return box3_lookup_rockets(scheme, mode, range);
        case LSG_HAM_AIR3D: return box3_lookup_air3d(scheme, mode, range);
    }
    return nullptr;
}

bool kernel_choice(const char* name) {
    const char* e = std::getenv("LSG_KERNEL");
    return e && std::string(e) == name;
}

bool pdl_enabled() {
    const char* e = std::getenv("LSG_PDL");
    return !(e && std::string(e) == "0");
}

bool force_generic() {
    const char* e = std::getenv("LSG_KERNEL");
    return e && std::string(e) == "generic";
}

EvalFn lookup_eval(int kind, int D) {
    switch (kind) {
        case LSG_HAM_LINEAR: return eval_lookup_linear(D);
        case LSG_HAM_NORMAL: return eval_lookup_normal(D);
        case LSG_HAM_ROTATION: return eval_lookup_rotation(D);
        case LSG_HAM_ROCKETS: return eval_lookup_rockets(D);
        case LSG_HAM_AIR3D: return eval_lookup_air3d(D);
        case LSG_HAM_DBLINT4: return eval_lookup_dblint4(D);
        case LSG_HAM_DUBINS6: return eval_lookup_dubins6(D);
    }
    return nullptr;
}

AlphaFn lookup_alpha(int kind) {
    switch (kind) {
        case LSG_HAM_LINEAR: return alpha_lookup_linear();
        case LSG_HAM_NORMAL: return alpha_lookup_normal();
        case LSG_HAM_ROTATION: return alpha_lookup_rotation();
        case LSG_HAM_ROCKETS: return alpha_lookup_rockets();
        case LSG_HAM_AIR3D: return alpha_lookup_air3d();
        case LSG_HAM_DBLINT4: return alpha_lookup_dblint4();
        case LSG_HAM_DUBINS6: return alpha_lookup_dubins6();
    }
    return nullptr;
}

// Grid dimension each kind requires (0: any); mirrors the reference's
// rocket_hamiltonian dimension check (reachability.cpp:22-25).
int kind_dim(int kind) {
    switch (kind) {
        case LSG_HAM_ROTATION: return 2;
        case LSG_HAM_ROCKETS: return 3;
        case LSG_HAM_AIR3D: return 3;
        case LSG_HAM_DBLINT4: return 4;
        case LSG_HAM_DUBINS6: return 6;
    }
    return 0;
}

// Whether a kind's Hamiltonian and dissipation bound are independent of t.
// The reference evaluates alpha at every stage time (hamiltonian.cpp:44-56);
// the device computes it once per solver and plans a leg's dt schedule up
// front, which is exact only for time-invariant kinds.  Every device kind is;
// a time-dependent kind must recompute alpha per stage time instead, and
// ensure_alpha refuses it until it does.
bool kind_time_invariant(int kind) {
    switch (kind) {
        case LSG_HAM_LINEAR:
        case LSG_HAM_ROTATION:
        case LSG_HAM_ROCKETS:
        case LSG_HAM_AIR3D:
        case LSG_HAM_DBLINT4:
        case LSG_HAM_DUBINS6:
        case LSG_HAM_NORMAL: return true;
    }
    return false;
}

unsigned trig_dims(int kind) {
    switch (kind) {
        case LSG_HAM_ROCKETS: return 1u << 2;
        case LSG_HAM_AIR3D: return 1u << 2;
        case LSG_HAM_DUBINS6: return (1u << 2) | (1u << 5);
    }
    return 0u;
}

}  // namespace

// ---- solver --------------------------------------------------------------------

struct Slab {
    int z0 = 0, nz = 0;
    long long nodes = 0;
    March3 m3{};       // 2.5-D tiling of this slab (3-D grids)
    dim3 m3_grid;
    CUtensorMap tmu[3], tmv[3];  // march3_tma_kernel: tile box / v0 box over each buffer
    DevBuf buf[3];
    double* f[3] = {nullptr, nullptr, nullptr};  // plane 0 of each buffer
};

struct lsg_solver {
    lsg_ctx* ctx = nullptr;
    lsg_grid g{};
    lsg_problem p{};
    int method = LSG_CFL3;
    int D = 0, W = 0;
    long long plane = 1;     // nodes per plane of the last axis
    long long total = 0;     // global node count
    int P = 1;               // slabs across the whole job
    int halo_w = 0;          // ghost planes per side (0 when the job has one slab)
    bool distributed = false;
    std::vector<Slab> slabs;
    DevBuf tables;
    const double* axis[kMaxDim] = {};
    const double* tcos[kMaxDim] = {};
    const double* tsin[kMaxDim] = {};
    LineConst lc[kMaxDim] = {};
    DevBuf dflags;  // unsigned[2]
    DevBuf dalpha;  // unsigned long long[8]: D keys, slot 7 = flags
    DevBuf drange;
    long long range_cap = 0;
    long long ring_next = 0;  // ring slot for lsg_solver_step
    double alpha[kMaxDim] = {};
    bool alpha_done = false;
    unsigned alpha_flags = 0;
    double bound = 0.0;
    StageFn fn[3] = {nullptr, nullptr, nullptr};
    March3Fn m3fn[3][2] = {};  // [mode][with v-range reduction]
    March3TmaFn m3tfn[3][2] = {};  // TMA-fed variant (even rows; LSG_TMA=0 disables)
    MarchNFn mnfn[3][2] = {};      // 4-D..6-D tile-and-march kernel
    Box3Fn b3fn[3][2] = {};
    int m3_threads = 0;
    int m3_pitch = 0;
    int m3_slot = 0, m3_vslot = 0, m3_hmax = 0;  // march3_tma_kernel ring geometry
    int m3_per_sm = 1;
    int div31_mask = 3;  // LSG_DIV31: which divmod31 paths slab_params may enable (tests)
    size_t m3_smem = 0;
    std::string invalid;  // deferred invalid_argument (raised at the first term evaluation)
    int cur = 0;
    // halo planes of buffer b hold the neighbours' current boundary planes
    // (set by the exchange that follows each stage's boundary bands; cleared
    // whenever the field is written from outside a stage)
    bool halo_ok[3] = {false, false, false};
    bool pdl = true;  // programmatic dependent launch between stages (LSG_PDL=0 disables; read at creation)
    bool nvtx = false;  // NVTX range per stage / exchange / leg (LSG_NVTX=1; read at creation)
    // halos: overlap the exchange with the interior (bands first on a side
    // stream), or exchange before each stage's single launch (LSG_HALO_OVERLAP=0)
    bool overlap_halo = true;
    cudaStream_t comm = nullptr;  // halo-exchange stream (slabs only)
    cudaStream_t side = nullptr;  // boundary bands, concurrent with the interior (slabs only)
    cudaStream_t cin = nullptr, cout = nullptr;  // lsg_solver_step_host copy streams (created on first use)
    std::vector<cudaEvent_t> pipe_ev;
    cudaEvent_t ev_ready = nullptr, ev_halo = nullptr, ev_main = nullptr, ev_bnd = nullptr;
    ~lsg_solver() {
        if (comm) cudaStreamSynchronize(comm);  // halo traffic done before the buffers go back to the pool
        if (side) cudaStreamSynchronize(side);
        for (cudaStream_t st : {cin, cout})
            if (st) cudaStreamSynchronize(st);
        for (cudaEvent_t e : pipe_ev) cudaEventDestroy(e);
        for (cudaStream_t st : {cin, cout})
            if (st) cudaStreamDestroy(st);
        for (cudaEvent_t e : {ev_ready, ev_halo, ev_main, ev_bnd})
            if (e) cudaEventDestroy(e);
        if (side) cudaStreamDestroy(side);
        if (comm) cudaStreamDestroy(comm);
    }
};

namespace {

constexpr long long kRingSlots = 4096;
// per-step range slot: {~min key, max key, ~first zero code} (lsg_kernels.cuh block_range)
constexpr long long kRangeWords = 3;

void partition(int n, int P, int r, int* z0, int* nz) {
    const int base = n / P, rem = n % P;
    *nz = base + (r < rem ? 1 : 0);
    *z0 = r * base + std::min(r, rem);
}

std::unique_ptr<lsg_solver> make_solver(lsg_ctx* ctx, const lsg_grid* g, const lsg_problem* p, int method,
                                        int nslabs) {
    activate(ctx);
    check_grid(g);
    if (!p) fail(LSG_EINVAL, "term_lax_friedrichs: problem must provide ham_func and dissipation_bounds");
    if (method < LSG_CFL1 || method > LSG_CFL3) fail(LSG_EINVAL, "unknown integrator");
    auto s = std::make_unique<lsg_solver>();
    s->ctx = ctx;
    s->g = *g;
    s->p = *p;
    s->method = method;
    s->D = g->dim;
    s->W = ghost_width(p->scheme);
    s->distributed = ctx->nranks > 1 || ctx->dist_selftest;
    s->pdl = pdl_enabled();
    if (const char* e = std::getenv("LSG_NVTX")) s->nvtx = std::string(e) == "1";
    if (const char* e = std::getenv("LSG_DIV31")) s->div31_mask = std::atoi(e) & 3;
    s->P = s->distributed ? ctx->nranks : nslabs;
    s->total = node_count(g);
    for (int d = 0; d + 1 < s->D; ++d) s->plane *= g->counts[d];
    s->halo_w = (s->P > 1 || s->distributed) ? s->W : 0;
    if (s->halo_w) {
        // halo traffic and boundary bands sit on the critical path of the next
        // stage: their blocks go ahead of the interior's when SMs free up
        int lo_prio = 0, hi_prio = 0;
        CUDA_CHECK(cudaDeviceGetStreamPriorityRange(&lo_prio, &hi_prio));
        CUDA_CHECK(cudaStreamCreateWithPriority(&s->comm, cudaStreamNonBlocking, hi_prio));
        CUDA_CHECK(cudaEventCreateWithFlags(&s->ev_ready, cudaEventDisableTiming));
        CUDA_CHECK(cudaEventCreateWithFlags(&s->ev_halo, cudaEventDisableTiming));
        CUDA_CHECK(cudaStreamCreateWithPriority(&s->side, cudaStreamNonBlocking, hi_prio));
        CUDA_CHECK(cudaEventCreateWithFlags(&s->ev_main, cudaEventDisableTiming));
        CUDA_CHECK(cudaEventCreateWithFlags(&s->ev_bnd, cudaEventDisableTiming));
    }
    const int nlast = g->counts[s->D - 1];
    if (s->P > nlast) fail(LSG_EINVAL, "slab decomposition: more slabs than planes along the last axis");

    // kind / dimension / stencil-room checks are deferred to the first term
    // evaluation, where the reference raises them (reachability.cpp:22,
    // spatial_derivatives.cpp:40-47).
    if (lookup_alpha(p->kind) == nullptr)  // not a device Hamiltonian kind
        s->invalid = "term_lax_friedrichs: problem must provide ham_func and dissipation_bounds";
    else if (kind_dim(p->kind) && kind_dim(p->kind) != s->D)
        s->invalid = "hamiltonian: grid dimension does not match the problem kind";
    for (int d = 0; d < s->D && s->invalid.empty(); ++d)
        if (g->counts[d] < min_nodes(p->scheme))
            s->invalid = std::string(scheme_name(p->scheme)) + ": needs at least " +
                         std::to_string(min_nodes(p->scheme)) + " nodes along dim " + std::to_string(d);
    // kernel scheme id: the opt-in one-division WENO5 is a separate instantiation
    const int kscheme = (p->scheme == LSG_SCHEME_WENO5 && (p->options & LSG_OPT_WENO5_FAST)) ? WENO5F : p->scheme;
    if (s->invalid.empty())
        for (int m = 0; m < 3; ++m) {
            s->fn[m] = lookup_stage(p->kind, s->D, kscheme, m);
            if (!s->fn[m]) s->invalid = "hamiltonian: kind not available for this grid dimension";
        }

    if (s->invalid.empty() && s->D == 3 && kernel_choice("box3") &&
        static_cast<long long>(g->counts[0]) * g->counts[1] < (1LL << 31))
        for (int m = 0; m < 3; ++m)
            for (int r = 0; r < 2; ++r) s->b3fn[m][r] = lookup_box3(p->kind, kscheme, m, r == 1);
    // 2.5-D tiled kernel for 3-D grids (lsg_march3.cuh): TX x R tiles, two
    // x-adjacent nodes per thread, 256 threads per block.
    int TX = 0, R = 0;
    // 4-D..6-D grids: the tile-and-march kernel over their first three axes
    // (lsg_marchn.cuh, same tile shapes) where it measured faster than the
    // one-node-per-thread kernel — the fast WENO5 in 4-D (cfg3 81^4: 30.4 ->
    // 33.5 G); elsewhere the generic kernel's 4 blocks per SM win (cfg3 exact
    // 14.8 vs 14.0 G, cfg4 exact 9.1 vs 7.9 G, ENO3 22.1 vs 19.9 G).
    // LSG_KERNEL=marchn forces it wherever it is instantiated.
    const bool marchn_ok = s->invalid.empty() && s->D >= 4 && !force_generic() && !kernel_choice("box3") &&
                           lookup_marchn(p->kind, s->D, kscheme, 0, false) != nullptr &&
                           (kernel_choice("marchn") || (kscheme == WENO5F && s->D == 4));
    if (s->invalid.empty() && (s->D == 3 || marchn_ok) && !force_generic() && !s->b3fn[0][0]) {
        const int n0 = g->counts[0], n1 = g->counts[1];
        const int W = s->W;
        // tile shapes in order of preference: full rows (no x halo), then x
        // segments; the first that fits 256 threads and kMaxHalo halo slots
        // per thread wins (full rows of more than ~120 nodes leave too few
        // rows per tile for the halo budget)
        std::vector<std::pair<int, int>> shapes;
        if (n0 <= 256) {
            // where full rows fit, rows split in three even segments when they are
            // >= 32 wide and need no more tiles: fewer halo rows per node (101^3:
            // 34x15 instead of 102x5, 1.65 instead of 2.2 loaded values per
            // node, +2.8 % on the bench)
            const int tf = (n0 + 1) & ~1, rf = std::max(1, 256 / (tf / 2));
            const int t3 = (((n0 + 2) / 3) + 1) & ~1, r3 = std::max(1, 256 / (t3 / 2));
            const long long tiles_f = static_cast<long long>((n1 + rf - 1) / rf);
            const long long tiles_3 = static_cast<long long>((n0 + t3 - 1) / t3) * ((n1 + r3 - 1) / r3);
            const int thf = ((tf / 2 * std::min(rf, n1) + 31) / 32) * 32;
            const bool full_fits = 2 * W * std::min(tf, n0) + 2 * W * std::min(rf, n1) <= kMaxHalo * thf;
            if (full_fits && t3 >= 32 && tiles_3 <= tiles_f) shapes.emplace_back(t3, r3);
            shapes.emplace_back(tf, rf);
        }
        shapes.emplace_back(32, 16);
        shapes.emplace_back(64, 8);
        if (const char* e = std::getenv("LSG_M3_TX")) {  // tuning override
            const int tx = std::max(2, std::atoi(e) & ~1);
            shapes.insert(shapes.begin(), {tx, std::max(1, 256 / (tx / 2))});
        }
        int threads = 0, halo = 0;
        bool fits = false;
        for (const auto& sh : shapes) {
            TX = sh.first;
            R = sh.second;
            if (const char* e = std::getenv("LSG_M3_R")) R = std::max(1, std::atoi(e));
            R = std::min(R, n1);
            threads = ((TX / 2 * R + 31) / 32) * 32;
            halo = 2 * W * std::min(TX, n0) + 2 * W * R;
            if (threads <= 256 && halo <= kMaxHalo * threads) {
                fits = true;
                break;
            }
        }
        if (fits && TX == 32 && R == std::min(16, n1) && !std::getenv("LSG_M3_TX") && !std::getenv("LSG_M3_R")) {
            // segment territory: a segment width of 28-64 whose tile count fits
            // the 148 x 2 block slots strictly better under the z-chunk model
            // used below (200^3: 30x17, 84 tiles in 7-plane chunks instead of 91
            // tiles in 67-plane chunks, +11 %); ties keep 32x16
            const int nzm = std::max(1, g->counts[2] / std::max(1, s->P));
            auto cost_of = [&](int tx, int r) {
                const int nt = ((n0 + tx - 1) / tx) * ((n1 + r - 1) / r);
                double best = 1e300;
                for (int nzc = 1; nzc <= nzm; ++nzc) {
                    const int chunk = (nzm + nzc - 1) / nzc;
                    const double waves = std::ceil(static_cast<double>(nt) * nzc / (148.0 * 2));
                    best = std::min(best, waves * (chunk + 0.5 * W + 1.0));
                }
                return best;
            };
            double best = cost_of(32, R);
            for (int tx = 28; tx <= 64; tx += 2) {
                const int r = std::min(256 / (tx / 2), n1);
                const int th = ((tx / 2 * r + 31) / 32) * 32;
                if (th > 256 || 2 * W * std::min(tx, n0) + 2 * W * r > kMaxHalo * th) continue;
                const double c = cost_of(tx, r);
                if (c < best * (1.0 - 1e-9)) {
                    best = c;
                    TX = tx;
                    R = r;
                    threads = th;
                }
            }
        }
        const long long padded_nodes = static_cast<long long>(g->counts[2] + 2 * W) * n0 * n1;
        if (fits && marchn_ok) {
            bool all = true;
            for (int m = 0; m < 3; ++m)
                for (int r = 0; r < 2; ++r) {
                    s->mnfn[m][r] = lookup_marchn(p->kind, s->D, kscheme, m, r == 1);
                    all = all && s->mnfn[m][r];
                }
            if (all) {
                s->m3_threads = threads;
                const int Wr = s->W, SHr = Wr & 1, XWr = (2 * Wr + 2 + SHr + 1) & ~1;
                s->m3_pitch = (TX + XWr - 2 + 1) & ~1;
                const int NB = 2 * Wr + 1 + 2, NV = 3;  // RingShape<W>
                s->m3_smem = sizeof(double) * static_cast<size_t>(NB * s->m3_pitch * (R + 2 * Wr) + NV * TX * R);
                for (int m = 0; m < 3; ++m)
                    for (int r = 0; r < 2; ++r)
                        CUDA_CHECK(cudaFuncSetAttribute(reinterpret_cast<const void*>(s->mnfn[m][r]),
                                                        cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                        static_cast<int>(s->m3_smem)));
                int per_sm = 0;
                CUDA_CHECK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(
                    &per_sm, reinterpret_cast<const void*>(s->mnfn[2][1]), threads, s->m3_smem));
                s->m3_per_sm = std::max(1, per_sm);
            } else {
                for (auto& fm : s->mnfn) fm[0] = fm[1] = nullptr;
            }
        } else if (fits && s->D == 3 && padded_nodes < (1LL << 31) - 1) {
            bool all = true;
            for (int m = 0; m < 3; ++m)
                for (int r = 0; r < 2; ++r) {
                    s->m3fn[m][r] = lookup_march3(p->kind, kscheme, m, r == 1);
                    all = all && s->m3fn[m][r];
                }
            if (all) {
                s->m3_threads = threads;
                const int Wr = s->W, SHr = Wr & 1, XWr = (2 * Wr + 2 + SHr + 1) & ~1;
                s->m3_pitch = (TX + XWr - 2 + 1) & ~1;
                const int NB = 2 * Wr + 1 + 2, NV = 3;  // RingShape<W>
                s->m3_smem = sizeof(double) * static_cast<size_t>(NB * s->m3_pitch * (R + 2 * Wr) + NV * TX * R);
                if (s->m3_smem > 48 * 1024)
                    for (int m = 0; m < 3; ++m)
                        for (int r = 0; r < 2; ++r)
                            CUDA_CHECK(cudaFuncSetAttribute(reinterpret_cast<const void*>(s->m3fn[m][r]),
                                                            cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                            static_cast<int>(s->m3_smem)));
                // TMA-fed tiles where rows are 16-byte multiples and the boxes fit.
                // WENO5 runs the y pass (march3_tma_kernel): one item of two rows
                // per thread, so R is made even (one row less) where needed
                const char* te = std::getenv("LSG_TMA");
                const bool yp = kscheme >= WENO5;
                int Rt = R, tht = threads;
                if (yp && Rt % 2 == 1 && Rt > 1) {
                    Rt -= 1;
                    tht = ((TX / 2 * Rt + 31) / 32) * 32;
                }
                const bool yp_ok = !yp || (Rt % 2 == 0 && TX * Rt <= 2 * tht &&
                                           2 * Wr * std::min(TX, n0) + 2 * Wr * Rt <= kMaxHalo * tht);
                const int rows_box = Rt + 2 * Wr;
                if (!(te && std::string(te) == "0") && yp_ok && n0 % 2 == 0 && s->m3_pitch <= 256 &&
                    rows_box <= 256 && TX <= 256 && Rt <= 256 && encode_tiled()) {
                    bool allt = true;
                    for (int m = 0; m < 3; ++m)
                        for (int r = 0; r < 2; ++r) {
                            s->m3tfn[m][r] = lookup_march3_tma(p->kind, kscheme, m, r == 1);
                            allt = allt && s->m3tfn[m][r];
                        }
                    if (allt) {
                        R = Rt;
                        threads = tht;
                        s->m3_threads = threads;
                        s->m3_slot = ((s->m3_pitch * rows_box + 15) / 16) * 16;
                        s->m3_vslot = ((TX * R + 15) / 16) * 16;
                        s->m3_hmax = 2 * Wr * (TX + R);
                        // ring depth of march3_tma_kernel (TmaDepth in lsg_march3.cuh): planes in flight
                        const int Dt = kscheme == WENO5 ? 1 : 2, NBt = 2 * Wr + 1 + Dt, NVt = Dt + 1;
                        s->m3_smem = sizeof(double) * static_cast<size_t>(NBt * s->m3_slot + NVt * s->m3_vslot +
                                                                          (Dt + 1) * s->m3_hmax +
                                                                          (yp ? 4 * TX * R : 0) +              // y-pass buffers
                                                                          (kscheme == WENO5F ? 4 * threads : 0)) +  // z-pair slots
                                     sizeof(unsigned long long) * NBt + 128;  // + alignment slack
                        for (int m = 0; m < 3; ++m)
                            for (int r = 0; r < 2; ++r)
                                CUDA_CHECK(cudaFuncSetAttribute(reinterpret_cast<const void*>(s->m3tfn[m][r]),
                                                                cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                                static_cast<int>(s->m3_smem)));
                    } else {
                        for (auto& fm : s->m3tfn) fm[0] = fm[1] = nullptr;
                    }
                }
                int per_sm = 0;
                CUDA_CHECK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(
                    &per_sm,
                    s->m3tfn[2][1] ? reinterpret_cast<const void*>(s->m3tfn[2][1])
                                   : reinterpret_cast<const void*>(s->m3fn[2][1]),
                    threads, s->m3_smem));
                s->m3_per_sm = std::max(1, per_sm);
            } else {
                for (auto& fm : s->m3fn) fm[0] = fm[1] = nullptr;
            }
        }
    }

    // halo mode: overlapped (bands, then the exchange concurrent with the
    // interior) by default; LSG_HALO_OVERLAP=0 exchanges before each stage's
    // single launch instead (measured equal within 1 % at 512^3 per rank on
    // the one-rank NCCL branch)
    {
        s->overlap_halo = true;
        if (const char* e = std::getenv("LSG_HALO_OVERLAP")) s->overlap_halo = std::string(e) != "0";
    }

    // slabs
    const int first = s->distributed ? ctx->rank : 0;
    const int count = s->distributed ? 1 : s->P;
    const int nbuf = method == LSG_CFL3 ? 3 : 2;
    for (int r = first; r < first + count; ++r) {
        Slab sl;
        partition(nlast, s->P, r, &sl.z0, &sl.nz);
        if (s->P > 1 && sl.nz < s->W)
            fail(LSG_EINVAL, "slab decomposition: each slab needs at least " + std::to_string(s->W) + " planes");
        sl.nodes = static_cast<long long>(sl.nz) * s->plane;
        if (s->mnfn[0][0]) {
            // tiles x outer indices x z-chunks of axis 2: enough blocks for >= 4 waves
            const int ntx = (g->counts[0] + TX - 1) / TX, nty = (g->counts[1] + R - 1) / R;
            long long outer = sl.nz;
            for (int d = 3; d + 1 < s->D; ++d) outer *= g->counts[d];
            const long long blocks = static_cast<long long>(ntx) * nty * outer;
            const long long want = 4LL * 148 * s->m3_per_sm;
            int nzc = static_cast<int>(std::min<long long>(std::max<long long>(1, (want + blocks - 1) / blocks),
                                                           std::max(1, g->counts[2] / 8)));
            if (const char* e = std::getenv("LSG_M3_CHUNK")) {
                const int chunk = std::max(1, std::min(g->counts[2], std::atoi(e)));
                nzc = (g->counts[2] + chunk - 1) / chunk;
            }
            if (std::getenv("LSG_M3_VERBOSE"))
                std::fprintf(stderr, "marchn D=%d: TX=%d R=%d tiles=%d outer=%lld chunks=%d blocks/SM=%d smem=%zu\n",
                             s->D, TX, R, ntx * nty, outer, nzc, s->m3_per_sm, s->m3_smem);
            sl.m3 = March3{TX, R, ntx, nzc, s->m3_pitch, 0, 0, 0};
            sl.m3_grid = dim3(static_cast<unsigned>(ntx * nty), static_cast<unsigned>(nzc));
        }
        if (s->m3fn[0][0]) {
            // tiles x z-chunks: minimise waves * (planes per chunk + warm-up) over 148 SMs
            const int ntx = (g->counts[0] + TX - 1) / TX, nty = (g->counts[1] + R - 1) / R;
            const int nt = ntx * nty;
            double best = 1e300;
            int best_nzc = 1;
            for (int nzc = 1; nzc <= sl.nz; ++nzc) {  // balanced split: chunks of ceil / floor(nz / nzc)
                const int chunk = (sl.nz + nzc - 1) / nzc;
                const double waves = std::ceil(static_cast<double>(nt) * nzc / (148.0 * s->m3_per_sm));
                const double cost = waves * (chunk + 0.5 * s->W + 1.0);
                if (cost < best + 1e-9) {  // ties: more, shorter chunks balance the SMs better
                    best = cost;
                    best_nzc = nzc;
                }
            }
            int nzc = best_nzc;
            // chunks of at most 64 planes: the wave model counts whole waves of
            // equal blocks, but finer chunks let the block scheduler even out
            // the slower border tiles (512^3, 4 -> 8 chunks: exact WENO5 +0.7 %,
            // ENO3 +1.3 %, fast WENO5 +1 %)
            nzc = std::max(nzc, (sl.nz + 63) / 64);
            if (const char* e = std::getenv("LSG_M3_CHUNK")) {  // planes per chunk (tuning override)
                const int chunk = std::max(1, std::min(sl.nz, std::atoi(e)));
                nzc = (sl.nz + chunk - 1) / chunk;
            }
            if (std::getenv("LSG_M3_VERBOSE"))
                std::fprintf(stderr, "march3%s: TX=%d R=%d tiles=%d chunks=%d blocks/SM=%d smem=%zu threads=%d\n",
                             s->m3tfn[0][0] ? " (TMA)" : "", TX, R, nt, nzc, s->m3_per_sm, s->m3_smem, s->m3_threads);
            sl.m3 = March3{TX, R, ntx, nzc, s->m3_pitch, s->m3_slot, s->m3_vslot, s->m3_hmax};
            sl.m3_grid = dim3(static_cast<unsigned>(nt), static_cast<unsigned>(nzc));
        }
        const long long padded = static_cast<long long>(sl.nz + 2 * s->halo_w) * s->plane;
        for (int b = 0; b < nbuf; ++b) {
            sl.buf[b].alloc(sizeof(double) * static_cast<size_t>(padded), ctx->stream);
            sl.f[b] = sl.buf[b].as<double>() + static_cast<long long>(s->halo_w) * s->plane;
            if (s->m3tfn[0][0]) {
                const int nzp = sl.nz + 2 * s->halo_w;
                sl.tmu[b] = tensor_map_3d(sl.buf[b].as<double>(), g->counts[0], g->counts[1], nzp, s->m3_pitch,
                                          sl.m3.R + 2 * s->W);
                sl.tmv[b] = tensor_map_3d(sl.buf[b].as<double>(), g->counts[0], g->counts[1], nzp, sl.m3.TX, sl.m3.R);
            }
        }
        s->slabs.push_back(std::move(sl));
    }

    // coordinate tables (grid.cpp:50) and host-libm trig tables
    std::vector<double> host;
    std::vector<size_t> ax_off(s->D), c_off(s->D, 0), s_off(s->D, 0);
    const unsigned tmask = trig_dims(p->kind);
    for (int d = 0; d < s->D; ++d) {
        const double dx = spacing(g, d);
        ax_off[d] = host.size();
        for (int i = 0; i < g->counts[d]; ++i) host.push_back(g->mins[d] + static_cast<double>(i) * dx);
    }
    for (int d = 0; d < s->D; ++d) {
        if (!(tmask & (1u << d))) continue;
        c_off[d] = host.size();
        for (int i = 0; i < g->counts[d]; ++i) host.push_back(std::cos(host[ax_off[d] + i]));
        s_off[d] = host.size();
        for (int i = 0; i < g->counts[d]; ++i) host.push_back(std::sin(host[ax_off[d] + i]));
    }
    s->tables.alloc(sizeof(double) * host.size(), ctx->stream);
    CUDA_CHECK(cudaMemcpyAsync(s->tables.p, host.data(), sizeof(double) * host.size(), cudaMemcpyHostToDevice,
                               ctx->stream));
    const double* base = s->tables.as<double>();
    for (int d = 0; d < s->D; ++d) {
        s->axis[d] = base + ax_off[d];
        if (tmask & (1u << d)) {
            s->tcos[d] = base + c_off[d];
            s->tsin[d] = base + s_off[d];
        }
        s->lc[d] = line_const(g, d);
    }
    s->dflags.alloc(sizeof(unsigned) * 2, ctx->stream);
    s->dalpha.alloc(sizeof(unsigned long long) * 8, ctx->stream);
    CUDA_CHECK(cudaMemsetAsync(s->dflags.p, 0, s->dflags.bytes, ctx->stream));
    s->drange.alloc(sizeof(unsigned long long) * kRangeWords * kRingSlots, ctx->stream);
    s->range_cap = kRingSlots;
    CUDA_CHECK(cudaMemsetAsync(s->drange.p, 0, s->drange.bytes, ctx->stream));
    CUDA_CHECK(cudaStreamSynchronize(ctx->stream));  // buffers usable from any stream from here on
    return s;
}

// The stateless reference-facing calls (term_lax_friedrichs, integrate,
// solve_brt) rebuild nothing when called again on the same grid, problem and
// integrator: the context keeps the last solver (device fields, axis/trig
// tables, alpha) keyed on the descriptors' bytes and the kernel-selection
// environment.  LSG_CALL_CACHE=0 disables it.
std::string solver_key(const lsg_grid* g, const lsg_problem* p, int method) {
    std::string k;
    auto put = [&k](const void* x, size_t n) { k.append(static_cast<const char*>(x), n); };
    put(&g->dim, sizeof g->dim);
    const int D = std::max(0, std::min(g->dim, kMaxDim));
    put(g->counts, sizeof(int) * D);
    put(g->mins, sizeof(double) * D);
    put(g->maxs, sizeof(double) * D);
    put(&g->periodic_mask, sizeof g->periodic_mask);
    put(&p->kind, sizeof p->kind);
    put(&p->scheme, sizeof p->scheme);
    put(&p->direction, sizeof p->direction);
    put(&p->restrict_update, sizeof p->restrict_update);
    put(&p->options, sizeof p->options);
    put(p->params, sizeof p->params);
    put(&method, sizeof method);
    for (const char* e : {"LSG_KERNEL", "LSG_M3_R", "LSG_M3_CHUNK", "LSG_DIV31", "LSG_PDL"}) {
        const char* v = std::getenv(e);
        k += '|';
        if (v) k += v;
    }
    return k;
}

void drop_cached(lsg_ctx* ctx) noexcept {  // also runs from a scope guard: never throws
    if (ctx->cached) {
        cudaStreamSynchronize(ctx->stream);
        delete ctx->cached;
    }
    ctx->cached = nullptr;
    ctx->cached_key.clear();
}

lsg_solver* cached_solver(lsg_ctx* ctx, const lsg_grid* g, const lsg_problem* p, int method) {
    activate(ctx);
    check_grid(g);
    if (!p) fail(LSG_EINVAL, "term_lax_friedrichs: problem must provide ham_func and dissipation_bounds");
    const char* off = std::getenv("LSG_CALL_CACHE");
    const bool enabled = !(off && std::string(off) == "0");
    std::string key = solver_key(g, p, method);
    if (enabled && ctx->cached && ctx->cached_key == key) {
        ctx->cached->cur = 0;
        return ctx->cached;
    }
    drop_cached(ctx);  // release its device memory before allocating the next
    ctx->cached = make_solver(ctx, g, p, method, 1).release();
    // large solvers are not kept: their buffers would crowd out the caller's own
    // allocations (CallCache drops them when the call returns)
    long long max_bytes = 2LL << 30;
    if (const char* e = std::getenv("LSG_CALL_CACHE_MAX_BYTES")) max_bytes = std::atoll(e);
    const long long bytes = static_cast<long long>(sizeof(double)) * ctx->cached->total * (method == LSG_CFL3 ? 3 : 2);
    ctx->cached_key = (enabled && bytes <= max_bytes) ? std::move(key) : std::string("\x01not cached");
    return ctx->cached;
}

// Scope guard of a stateless call: a solver that is not to be kept (caching
// disabled or too large) is released when the call returns, also on errors.
struct CallCache {
    lsg_ctx* ctx;
    ~CallCache() {
        if (ctx && ctx->cached && ctx->cached_key.rfind("\x01", 0) == 0) drop_cached(ctx);
    }
};

// Build a solver; when the device is out of memory and the context still
// holds a cached stateless-call solver, release that and retry once.
std::unique_ptr<lsg_solver> make_solver_retry(lsg_ctx* ctx, const lsg_grid* g, const lsg_problem* p, int method,
                                              int nslabs) {
    try {
        return make_solver(ctx, g, p, method, nslabs);
    } catch (const Error& e) {
        if (e.code != LSG_ENOMEM || !ctx || !ctx->cached) throw;
        drop_cached(ctx);
        return make_solver(ctx, g, p, method, nslabs);
    }
}

// Before a collective on the main stream: the halo exchange last issued on the
// communication stream (the one that follows a stage's boundary bands) is
// complete, so the communicator's operations run in one order on every rank
// whatever the library's cross-stream ordering.
void join_comm(lsg_solver* s) {
    if (s->comm && s->ev_halo) CUDA_CHECK(cudaStreamWaitEvent(s->ctx->stream, s->ev_halo, 0));
}

void ensure_range(lsg_solver* s, long long nslots) {
    if (s->range_cap < nslots) {
        s->drange.alloc(sizeof(unsigned long long) * kRangeWords * static_cast<size_t>(nslots), s->ctx->stream);
        s->range_cap = nslots;
    }
    CUDA_CHECK(cudaMemsetAsync(s->drange.p, 0, sizeof(unsigned long long) * kRangeWords * static_cast<size_t>(nslots),
                               s->ctx->stream));
    s->ring_next = 0;
}

// Global Lax-Friedrichs alpha (hamiltonian.cpp:44-56) and the CFL bound (:68-71).
void ensure_alpha(lsg_solver* s) {
    if (s->alpha_done) return;
    if (!s->invalid.empty()) fail(LSG_EINVAL, s->invalid);
    if (!kind_time_invariant(s->p.kind))
        fail(LSG_EINVAL, "hamiltonian: time-dependent kinds need per-stage alpha (not implemented)");
    lsg_ctx* ctx = s->ctx;
    CUDA_CHECK(cudaMemsetAsync(s->dalpha.p, 0, s->dalpha.bytes, ctx->stream));
    AlphaFn fn = lookup_alpha(s->p.kind);
    for (const Slab& sl : s->slabs) {
        AlphaParams A{};
        A.n_local = sl.nodes;
        A.D = s->D;
        for (int d = 0; d < s->D; ++d) {
            A.n[d] = d == s->D - 1 ? sl.nz : s->g.counts[d];
            A.axis[d] = s->axis[d];
            A.tcos[d] = s->tcos[d];
            A.tsin[d] = s->tsin[d];
        }
        A.z0 = sl.z0;
        A.trig_dim = s->p.kind == LSG_HAM_ROCKETS || s->p.kind == LSG_HAM_AIR3D ? 2 : -1;
        std::memcpy(A.hp, s->p.params, sizeof A.hp);
        A.out = s->dalpha.as<unsigned long long>();
        A.flags = reinterpret_cast<unsigned*>(s->dalpha.as<unsigned long long>() + 7);
        void* args[] = {&A};
        CUDA_CHECK(cudaLaunchKernel(reinterpret_cast<const void*>(fn), dim3((unsigned)((sl.nodes + 255) / 256)),
                                    dim3(256), args, 0, ctx->stream));
        ctx->note_launch();
    }
    if (s->distributed) {
        join_comm(s);
        NCCL_CHECK(ncclAllReduce(s->dalpha.p, s->dalpha.p, 8, ncclUint64, ncclMax, ctx->comm, ctx->stream));
    }
    unsigned long long keys[8];
    CUDA_CHECK(cudaMemcpyAsync(keys, s->dalpha.p, sizeof keys, cudaMemcpyDeviceToHost, ctx->stream));
    CUDA_CHECK(cudaStreamSynchronize(ctx->stream));
    for (int d = 0; d < s->D; ++d) std::memcpy(&s->alpha[d], &keys[d], sizeof(double));
    s->alpha_flags = static_cast<unsigned>(keys[7]);
    double speed = 0.0;
    for (int d = 0; d < s->D; ++d) speed += s->alpha[d] / spacing(&s->g, d);
    s->bound = speed > 0.0 ? 1.0 / speed : std::numeric_limits<double>::infinity();
    s->alpha_done = true;
}

void check_alpha_valid(lsg_solver* s) {
    ensure_alpha(s);
    if (s->alpha_flags & FLAG_BOUND_INVALID)
        fail(LSG_ENUMERIC, "term_lax_friedrichs: dissipation bound must be finite and non-negative");
}

// The halo messages of one rank, in issue order (lsg_halo_plan): every rank
// sends its top W planes up, then its bottom W planes down, then receives the
// lower ghost planes from below and the upper ones from above, so per peer
// pair the messages match in issue order even for a 2-rank periodic ring.
struct HaloMsg {
    int kind;  // 0 send, 1 recv
    int peer;
    int plane;  // first plane, relative to the slab's plane 0 (ghost planes negative / >= nz)
    int count;  // planes
};
int halo_plan(int n, int nranks, int rank, int w, bool periodic, HaloMsg* out) {
    int z0 = 0, nz = 0;
    partition(n, nranks, rank, &z0, &nz);
    const int lo = rank > 0 ? rank - 1 : (periodic ? nranks - 1 : -1);
    const int hi = rank < nranks - 1 ? rank + 1 : (periodic ? 0 : -1);
    int k = 0;
    if (hi >= 0) out[k++] = {0, hi, nz - w, w};
    if (lo >= 0) out[k++] = {0, lo, 0, w};
    if (lo >= 0) out[k++] = {1, lo, -w, w};
    if (hi >= 0) out[k++] = {1, hi, nz, w};
    return k;
}

// Fill the ghost planes of buffer b: from the neighbour slabs (device copies
// in-process, NCCL send/recv across ranks); ring for a periodic last axis.
void exchange(lsg_solver* s, int b, cudaStream_t st) {
    if (s->halo_w == 0) return;
    NvtxRange nv(s->nvtx, "lsg halo exchange");
    lsg_ctx* ctx = s->ctx;
    const bool periodic = bc_of(&s->g, s->D - 1) == LSG_BC_PERIODIC;
    const long long w = s->halo_w;
    const size_t bytes = sizeof(double) * static_cast<size_t>(w * s->plane);
    if (!s->distributed) {
        const int P = s->P;
        for (int r = 0; r < P; ++r) {
            Slab& me = s->slabs[r];
            const int lo = r > 0 ? r - 1 : (periodic ? P - 1 : -1);
            const int hi = r < P - 1 ? r + 1 : (periodic ? 0 : -1);
            if (lo >= 0) {
                const Slab& o = s->slabs[lo];
                CUDA_CHECK(cudaMemcpyAsync(me.f[b] - w * s->plane, o.f[b] + (o.nz - w) * s->plane, bytes,
                                           cudaMemcpyDeviceToDevice, st));
            }
            if (hi >= 0) {
                const Slab& o = s->slabs[hi];
                CUDA_CHECK(cudaMemcpyAsync(me.f[b] + me.nz * s->plane, o.f[b], bytes, cudaMemcpyDeviceToDevice, st));
            }
        }
        return;
    }
    Slab& me = s->slabs[0];
    HaloMsg msg[4];
    const int nmsg = halo_plan(s->g.counts[s->D - 1], ctx->nranks, ctx->rank, static_cast<int>(w), periodic, msg);
    NCCL_CHECK(ncclGroupStart());
    for (int k = 0; k < nmsg; ++k) {
        double* p = me.f[b] + static_cast<long long>(msg[k].plane) * s->plane;
        const size_t cnt = static_cast<size_t>(msg[k].count) * static_cast<size_t>(s->plane);
        if (msg[k].kind == 0)
            NCCL_CHECK(ncclSend(p, cnt, ncclFloat64, msg[k].peer, ctx->comm, st));
        else
            NCCL_CHECK(ncclRecv(p, cnt, ncclFloat64, msg[k].peer, ctx->comm, st));
    }
    NCCL_CHECK(ncclGroupEnd());
}

// Geometry, tables, alpha, clamp and flags of one slab (what every stage of
// every kernel variant shares).
StageParams slab_params(lsg_solver* s, const Slab& sl) {
    const int D = s->D;
    StageParams P{};
    P.zlo = 0;
    P.zhi = sl.nz;
    P.plane = s->plane;
    P.n_local = sl.nodes;
    long long st = 1;
    for (int d = 0; d < D; ++d) {
        P.n[d] = d == D - 1 ? sl.nz : s->g.counts[d];
        P.inv_n[d] = 1.0 / P.n[d];
        if (P.n[d] >= 2) {
            int l = 0;
            while ((1LL << l) < P.n[d]) ++l;
            P.magic[d] = static_cast<unsigned>(((1ULL << (31 + l)) + P.n[d] - 1) / static_cast<unsigned long long>(P.n[d]));
            P.mshift[d] = l - 1;
        }
        P.stride[d] = st;
        st *= P.n[d];
        P.bc[d] = bc_of(&s->g, d);
        P.lc[d] = s->lc[d];
        P.alpha[d] = s->alpha[d];
        P.alpha_f[d] = s->alpha[d] * (s->lc[d].inv_dx * (1.0 / 6.0));
        P.axis[d] = s->axis[d];
        P.tcos[d] = s->tcos[d];
        P.tsin[d] = s->tsin[d];
    }
    bool all2 = true;
    for (int d = 0; d < D - 1; ++d) all2 = all2 && P.n[d] >= 2;
    if (all2) {  // divmod31 where the dividends fit 31 bits (lsg_device.cuh)
        P.div31 = ((sl.nodes <= (1LL << 31) ? 1 : 0) | ((sl.nodes - 1) / P.n[0] < (1LL << 31) ? 2 : 0)) & s->div31_mask;
    }
    P.z0 = sl.z0;
    P.nz_glob = s->g.counts[D - 1];
    P.halo = s->halo_w > 0 ? 1 : 0;
    P.restrict_update = s->p.restrict_update;
    P.direction = s->p.direction;
    std::memcpy(P.hp, s->p.params, sizeof P.hp);
    P.flags = s->dflags.as<unsigned>();
    return P;
}

// One stage kernel over the logical planes [zlo, zhi) of slab `sl` (planes at
// or past zsplit shifted by zskip) on `stream`.
void launch_planes(lsg_solver* s, Slab& sl, int mode, int ui, int vi, int oi, double dt, double c,
                   unsigned long long* range, int zlo, int zhi, int zsplit, int zskip, cudaStream_t stream,
                   int reserve_blocks = 0) {
    lsg_ctx* ctx = s->ctx;
    StageParams P = slab_params(s, sl);
    P.zlo = zlo;
    P.zhi = zhi;
    P.zsplit = zsplit;
    P.zskip = zskip;
    P.u = sl.f[ui];
    P.v0 = vi >= 0 ? sl.f[vi] : nullptr;
    P.out = sl.f[oi];
    P.dt = dt;
    P.c = c;
    P.range = range;
    if (s->b3fn[mode][0]) {
        void* args[] = {&P};
        const long long pl = s->plane;
        CUDA_CHECK(cudaLaunchKernel(reinterpret_cast<const void*>(s->b3fn[mode][range ? 1 : 0]),
                                    dim3(static_cast<unsigned>((pl + 255) / 256), static_cast<unsigned>(zhi - zlo)),
                                    dim3(256), args, 0, stream));
    } else if (s->mnfn[mode][0]) {
        March3 M = sl.m3;
        long long mid = 1;
        for (int d = 3; d + 1 < s->D; ++d) mid *= s->g.counts[d];
        const long long gx = static_cast<long long>(sl.m3_grid.x) * mid * (zhi - zlo);
        void* args[] = {&P, &M};
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(static_cast<unsigned>(gx), static_cast<unsigned>(M.nzc));
        cfg.blockDim = dim3(static_cast<unsigned>(s->m3_threads));
        cfg.dynamicSmemBytes = s->m3_smem;
        cfg.stream = stream;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        attr[0].val.programmaticStreamSerializationAllowed = s->pdl ? 1 : 0;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        CUDA_CHECK(cudaLaunchKernelExC(&cfg, reinterpret_cast<const void*>(s->mnfn[mode][range ? 1 : 0]), args));
    } else if (s->m3fn[mode][0]) {
        March3 M = sl.m3;
        if (zhi - zlo < sl.nz) {
            // a partial range (step_host chunks, a slab's interior): enough
            // chunks to fill one wave and keep chunks <= 64 planes, no more
            // than the full slab's and none under 3 planes (512^3 in 16-plane
            // step_host chunks: one chunk per tile, e2e 16.2 -> 16.7 G;
            // 101^3: 8 chunks; a 512^3 slab's interior: 8 chunks)
            const int R = zhi - zlo;
            const int tiles = static_cast<int>(sl.m3_grid.x);
            const int fill = (148 * s->m3_per_sm + tiles - 1) / tiles;
            M.nzc = std::max(1, std::min(std::max(fill, (R + 63) / 64), std::min(M.nzc, R / 3)));
        }
        if (reserve_blocks > 0 && 2 * reserve_blocks <= 148 * s->m3_per_sm) {
            // share one wave with a concurrent launch (the boundary bands) when
            // the bands are a small part of a wave; with many tiles they are not,
            // and the interior keeps its balanced chunks
            const int slots = 148 * s->m3_per_sm - reserve_blocks;
            M.nzc = std::max(1, std::min(M.nzc, slots / std::max(1, static_cast<int>(sl.m3_grid.x))));
        }
        if (zskip) M.nzc = 2;  // one chunk per band: none straddles the gap
        const dim3 grid(sl.m3_grid.x, static_cast<unsigned>(M.nzc));
        void* args[] = {&P, &M, &sl.tmu[ui], &sl.tmv[vi >= 0 ? vi : ui]};
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = grid;
        cfg.blockDim = dim3(static_cast<unsigned>(s->m3_threads));
        cfg.dynamicSmemBytes = s->m3_smem;
        cfg.stream = stream;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;  // PDL with the previous stage
        attr[0].val.programmaticStreamSerializationAllowed = s->pdl ? 1 : 0;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        const void* fn = s->m3tfn[mode][0] ? reinterpret_cast<const void*>(s->m3tfn[mode][range ? 1 : 0])
                                           : reinterpret_cast<const void*>(s->m3fn[mode][range ? 1 : 0]);
        CUDA_CHECK(cudaLaunchKernelExC(&cfg, fn, args));
    } else {
        void* args[] = {&P};
        const long long n = static_cast<long long>(zhi - zlo) * s->plane;
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3((unsigned)((n + 255) / 256));
        cfg.blockDim = dim3(256);
        cfg.stream = stream;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        attr[0].val.programmaticStreamSerializationAllowed = s->pdl ? 1 : 0;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        CUDA_CHECK(cudaLaunchKernelExC(&cfg, reinterpret_cast<const void*>(s->fn[mode]), args));
    }
    ctx->note_launch();
}

// One stage kernel per slab on `stream`; `part` selects the planes:
// 0: all planes; 1: interior planes [W, nz-W) that need no ghost planes;
// 2: both boundary bands [0, W) and [nz-W, nz) in one launch (logical planes
// [0, 2W) with a gap of nz-2W planes after W).
void launch_stage(lsg_solver* s, int mode, int ui, int vi, int oi, double dt, double c, unsigned long long* range,
                  int part, cudaStream_t stream) {
    for (Slab& sl : s->slabs) {
        int zlo = 0, zhi = sl.nz, zsplit = 0, zskip = 0;
        const int W = s->halo_w;
        if (part == 1) {
            zlo = W, zhi = sl.nz - W;
            if (zhi <= zlo) continue;
        } else if (part == 2 && sl.nz > 2 * W) {
            zhi = 2 * W, zsplit = W, zskip = sl.nz - 2 * W;
        }
        // the interior runs beside the bands' launch (two chunks per tile)
        const int reserve = part == 1 ? 2 * static_cast<int>(sl.m3_grid.x) : 0;
        launch_planes(s, sl, mode, ui, vi, oi, dt, c, range, zlo, zhi, zsplit, zskip, stream, reserve);
    }
}

// One fused stage over every slab.  Without halos: one launch.  With halos
// (several slabs or ranks):
//   side stream: the boundary bands (one launch), once the main stream's
//                previous stage and the exchange of u's halo are done;
//   comm stream: the exchange of the bands' fresh output planes (the next
//                stage's halo), as soon as the bands finish;
//   main stream: the interior planes, concurrently, then a join on the bands.
// So the halo traffic overlaps the interior and the next stage finds it done.
// A field written from outside a stage (upload, device copy, initial shape)
// has no valid halo and is exchanged before its first stage.
void run_stage(lsg_solver* s, int mode, int ui, int vi, int oi, double dt, double c, unsigned long long* range) {
    lsg_ctx* ctx = s->ctx;
    static const char* const names[3] = {"lsg term (TERM)", "lsg RK stage (EULER)", "lsg RK stage (COMBINE)"};
    NvtxRange nv(s->nvtx, names[mode]);
    if (s->halo_w == 0) {
        launch_stage(s, mode, ui, vi, oi, dt, c, range, 0, ctx->stream);
        return;
    }
    auto exchange_after = [&](cudaEvent_t ev, cudaStream_t from, int b) {
        CUDA_CHECK(cudaEventRecord(ev, from));
        CUDA_CHECK(cudaStreamWaitEvent(s->comm, ev, 0));
        exchange(s, b, s->comm);
        CUDA_CHECK(cudaEventRecord(s->ev_halo, s->comm));
    };
    if (!s->overlap_halo) {  // large slabs: exchange u's halo, then one launch over all planes
        if (!s->halo_ok[ui]) {
            join_comm(s);
            exchange(s, ui, ctx->stream);
            s->halo_ok[ui] = true;
        }
        launch_stage(s, mode, ui, vi, oi, dt, c, range, 0, ctx->stream);
        s->halo_ok[oi] = false;
        return;
    }
    if (!s->halo_ok[ui]) {
        exchange_after(s->ev_ready, ctx->stream, ui);
        s->halo_ok[ui] = true;
    }
    CUDA_CHECK(cudaEventRecord(s->ev_main, ctx->stream));
    CUDA_CHECK(cudaStreamWaitEvent(s->side, s->ev_main, 0));
    CUDA_CHECK(cudaStreamWaitEvent(s->side, s->ev_halo, 0));
    launch_stage(s, mode, ui, vi, oi, dt, c, range, 2, s->side);
    if (mode != MODE_TERM && oi != ui) {
        exchange_after(s->ev_bnd, s->side, oi);  // the next stage's halo
        s->halo_ok[oi] = true;
    } else {
        CUDA_CHECK(cudaEventRecord(s->ev_bnd, s->side));
        s->halo_ok[oi] = false;
    }
    launch_stage(s, mode, ui, vi, oi, dt, c, range, 1, ctx->stream);
    CUDA_CHECK(cudaStreamWaitEvent(ctx->stream, s->ev_bnd, 0));
}

// One TVD-RK step (integrator.cpp:58-85); buffers: cur = v, the others scratch.
// ev (optional) receives stages+1 events: before the step and after each stage.
void enqueue_step(lsg_solver* s, double dt, unsigned long long* range, cudaEvent_t* ev = nullptr) {
    const int a = s->cur;
    cudaStream_t st = s->ctx->stream;
    auto mark = [&](int k) {
        if (ev) CUDA_CHECK(cudaEventRecord(ev[k], st));
    };
    mark(0);
    if (s->method == LSG_CFL1) {
        const int b = 1 - a;
        run_stage(s, MODE_EULER, a, -1, b, dt, 0.0, range);
        s->cur = b;
    } else if (s->method == LSG_CFL2) {
        const int b = 1 - a;
        run_stage(s, MODE_EULER, a, -1, b, dt, 0.0, nullptr);
        mark(1);
        run_stage(s, MODE_COMBINE, b, a, a, dt, 0.5, range);
    } else {
        const int b = (a + 1) % 3, c = (a + 2) % 3;
        run_stage(s, MODE_EULER, a, -1, b, dt, 0.0, nullptr);
        mark(1);
        run_stage(s, MODE_COMBINE, b, a, c, dt, 0.25, nullptr);
        mark(2);
        run_stage(s, MODE_COMBINE, c, a, a, dt, 2.0 / 3.0, range);
    }
    // the step ends when its last exchange (the next step's halo) has landed:
    // the main stream joins the communication stream, so an event recorded
    // after the step (bench timing, step_timed) covers the halo traffic too
    join_comm(s);
    mark(s->method + 1);
}

int stages_of(int method) { return method + 1; }

void check_options(const lsg_opts* o) {  // integrator.cpp:11-20
    if (!(o->cfl_factor > 0.0)) fail(LSG_EINVAL, "integrator: cfl_factor must be positive");
    if (!(o->max_step > 0.0)) fail(LSG_EINVAL, "integrator: max_step must be positive");
    if (!(o->termination_epsilon > 0.0)) fail(LSG_EINVAL, "integrator: termination_epsilon must be positive");
    for (size_t k = 1; k < o->n_checkpoint_times; ++k)
        if (o->checkpoint_times[k] < o->checkpoint_times[k - 1])
            fail(LSG_EINVAL, "integrator: checkpoint_times must be ascending");
}

lsg_opts default_opts() {
    lsg_opts o;
    o.cfl_factor = 0.32;
    o.max_step = std::numeric_limits<double>::infinity();
    o.termination_epsilon = 1e-6;
    o.checkpoint_times = nullptr;
    o.n_checkpoint_times = 0;
    return o;
}

double smin(double a, double b) { return (b < a) ? b : a; }  // std::min

// An invalid dissipation bound, reported as term_lax_friedrichs does: H is
// evaluated on the current field first and a non-finite H wins
// (hamiltonian.cpp:37-56).  One TERM stage into a scratch buffer.
[[noreturn]] void fail_bound_invalid(lsg_solver* s) {
    lsg_ctx* ctx = s->ctx;
    const int nbuf = s->method == LSG_CFL3 ? 3 : 2;
    CUDA_CHECK(cudaMemsetAsync(s->dflags.p, 0, sizeof(unsigned), ctx->stream));
    run_stage(s, MODE_TERM, s->cur, -1, (s->cur + 1) % nbuf, 0.0, 0.0, nullptr);
    if (s->distributed) {
        join_comm(s);
        NCCL_CHECK(ncclAllReduce(s->dflags.p, s->dflags.p, 1, ncclUint32, ncclMax, ctx->comm, ctx->stream));
    }
    unsigned flags = 0;
    CUDA_CHECK(cudaMemcpyAsync(&flags, s->dflags.p, sizeof flags, cudaMemcpyDeviceToHost, ctx->stream));
    CUDA_CHECK(cudaStreamSynchronize(ctx->stream));
    if (flags & FLAG_HAM_NONFINITE) fail(LSG_ENUMERIC, "term_lax_friedrichs: hamiltonian produced a non-finite value");
    fail(LSG_ENUMERIC, "term_lax_friedrichs: dissipation bound must be finite and non-negative");
}

// The dt schedule of one leg of run_cfl (integrator.cpp:22-97), host only:
// alpha and the CFL bound are v-independent, so every step's (t, dt) follows
// from (t0, tf, options) alone.  Validation errors are raised in the
// reference's order.
struct LegPlan {
    std::vector<lsg_steplog> log;
    double t_final = 0.0;
    bool collapsed = false;
    bool bound_invalid = false;  // raised by run_leg once H has been checked on the leg's field
};

LegPlan plan_leg(lsg_solver* s, double t0, double tf, const lsg_opts* opts_in) {
    const lsg_opts o = opts_in ? *opts_in : default_opts();
    check_options(&o);
    if (!std::isfinite(t0) || !std::isfinite(tf)) fail(LSG_EINVAL, "integrator: tspan must be finite");
    if (tf < t0) fail(LSG_EINVAL, "integrator: tspan must not be decreasing");
    LegPlan plan;
    plan.t_final = t0;
    if (tf == t0) return plan;
    const double eps_stop = o.termination_epsilon * std::abs(tf);
    double t = t0;
    if (!(tf - t > 0.0 && tf - t >= eps_stop)) return plan;
    // the first term evaluation validates the bounds, after H (run_leg)
    ensure_alpha(s);
    if (s->alpha_flags & FLAG_BOUND_INVALID) {
        plan.bound_invalid = true;
        return plan;
    }
    while (tf - t > 0.0 && tf - t >= eps_stop) {
        double target = tf;
        if (o.n_checkpoint_times) {
            const double* b = o.checkpoint_times;
            const double* e = b + o.n_checkpoint_times;
            const double* next = std::upper_bound(b, e, t);
            if (next != e && *next < tf) target = *next;
        }
        const double remaining = target - t;
        double dt = smin(remaining, o.max_step);
        dt = smin(dt, o.cfl_factor * s->bound);
        if (!(dt > 0.0)) {
            plan.collapsed = true;
            break;
        }
        const bool lands = dt == remaining;
        plan.log.push_back({t, dt, s->bound, 0.0, 0.0});
        t = lands ? target : t + dt;
    }
    plan.t_final = t;
    return plan;
}

// Run a planned leg on the device-resident field: every stage of every step
// enqueued back to back, one synchronisation at the end for the per-step v
// range and the error flags.
void run_leg(lsg_solver* s, LegPlan& plan) {
    NvtxRange nv(s->nvtx, "lsg leg (run_cfl)");
    if (plan.bound_invalid) fail_bound_invalid(s);
    std::vector<lsg_steplog>& log = plan.log;
    const bool collapsed = plan.collapsed;
    const long long nsteps = static_cast<long long>(log.size());
    lsg_ctx* ctx = s->ctx;
    CUDA_CHECK(cudaMemsetAsync(s->dflags.p, 0, sizeof(unsigned), ctx->stream));
    ensure_range(s, std::max<long long>(nsteps, 1));
    for (long long k = 0; k < nsteps; ++k)
        enqueue_step(s, log[k].dt, s->drange.as<unsigned long long>() + kRangeWords * k);
    unsigned flags = 0;
    if (s->distributed) {
        join_comm(s);
        NCCL_CHECK(ncclAllReduce(s->dflags.p, s->dflags.p, 1, ncclUint32, ncclMax, ctx->comm, ctx->stream));
        if (nsteps)  // both slots are max-reduced: {~min key, max key} per step
            NCCL_CHECK(ncclAllReduce(s->drange.p, s->drange.p, static_cast<size_t>(kRangeWords * nsteps), ncclUint64, ncclMax,
                                     ctx->comm, ctx->stream));
    }
    std::vector<unsigned long long> keys(static_cast<size_t>(kRangeWords * nsteps));
    CUDA_CHECK(cudaMemcpyAsync(&flags, s->dflags.p, sizeof(unsigned), cudaMemcpyDeviceToHost, ctx->stream));
    if (nsteps)
        CUDA_CHECK(cudaMemcpyAsync(keys.data(), s->drange.p, sizeof(unsigned long long) * keys.size(),
                                   cudaMemcpyDeviceToHost, ctx->stream));
    CUDA_CHECK(cudaStreamSynchronize(ctx->stream));
    if (flags & FLAG_HAM_NONFINITE)
        fail(LSG_ENUMERIC, "term_lax_friedrichs: hamiltonian produced a non-finite value");
    if (collapsed) fail(LSG_ENUMERIC, "integrator: step size collapsed to zero");
    for (long long k = 0; k < nsteps; ++k) {
        const unsigned long long* w = keys.data() + kRangeWords * k;
        double vmin = key_to_double(~w[0]), vmax = key_to_double(w[1]);
        // +-0 share a key; integrator.cpp:87-90 keeps the first of equal values,
        // i.e. the first zero in index order decides the sign (~w[2] = its code)
        const unsigned long long fz = ~w[2];
        if (fz != ~0ull) {
            const double zero = (fz & 1ull) ? -0.0 : 0.0;
            if (vmin == 0.0) vmin = zero;
            if (vmax == 0.0) vmax = zero;
        }
        log[k].v_min = vmin;
        log[k].v_max = vmax;
    }
}

// Step-log capacity check before any device work: LSG_ERANGE with the needed
// entry count in *n_steps, nothing modified (the caller retries).
void check_log_room(size_t need, const lsg_steplog* steps, size_t cap, size_t* n_steps) {
    if (steps && need > cap) {
        if (n_steps) *n_steps = need;
        fail(LSG_ERANGE, "step log capacity " + std::to_string(cap) + " too small: " + std::to_string(need) +
                             " entries needed");
    }
}

void copy_log(const std::vector<lsg_steplog>& log, lsg_steplog* out, size_t cap, size_t* n) {
    if (n) *n = log.size();
    if (out)
        for (size_t k = 0; k < log.size() && k < cap; ++k) out[k] = log[k];
}

void invalidate_halos(lsg_solver* s) {
    for (bool& h : s->halo_ok) h = false;
}

void upload(lsg_solver* s, const double* host, int b) {
    lsg_ctx* ctx = s->ctx;
    invalidate_halos(s);
    if (s->distributed) {
        const Slab& sl = s->slabs[0];
        CUDA_CHECK(cudaMemcpyAsync(sl.f[b], host, sizeof(double) * sl.nodes, cudaMemcpyHostToDevice, ctx->stream));
        return;
    }
    for (const Slab& sl : s->slabs)
        CUDA_CHECK(cudaMemcpyAsync(sl.f[b], host + static_cast<long long>(sl.z0) * s->plane,
                                   sizeof(double) * sl.nodes, cudaMemcpyHostToDevice, ctx->stream));
}

void download(lsg_solver* s, double* host, int b) {
    lsg_ctx* ctx = s->ctx;
    if (s->distributed) {
        const Slab& sl = s->slabs[0];
        CUDA_CHECK(cudaMemcpyAsync(host, sl.f[b], sizeof(double) * sl.nodes, cudaMemcpyDeviceToHost, ctx->stream));
    } else {
        for (const Slab& sl : s->slabs)
            CUDA_CHECK(cudaMemcpyAsync(host + static_cast<long long>(sl.z0) * s->plane, sl.f[b],
                                       sizeof(double) * sl.nodes, cudaMemcpyDeviceToHost, ctx->stream));
    }
    CUDA_CHECK(cudaStreamSynchronize(ctx->stream));
}

// Gather the slabs of a distributed field into global_host on rank 0 (the
// slab axis is the slowest, so the global column-major array is the slabs
// concatenated in rank order; reachability.cpp:160-170, snapshot.cpp:68-93).
// Each rank passes its slab as a device pointer (dev_local) or a host
// pointer (host_local).  Point-to-point NCCL in 1 GiB chunks through one
// device staging buffer; ranks other than 0 only send.  Collective.
void gather_to_root(lsg_ctx* ctx, const lsg_grid* g, const double* dev_local, const double* host_local,
                    double* global_host) {
    const int D = g->dim, P = ctx->nranks, me = ctx->rank;
    long long plane = 1;
    for (int d = 0; d + 1 < D; ++d) plane *= g->counts[d];
    const long long chunk = 1LL << 27;  // doubles (1 GiB)
    DevBuf stage;
    auto slab_of = [&](int r, long long* off, long long* n) {
        int z0 = 0, nz = 0;
        partition(g->counts[D - 1], P, r, &z0, &nz);
        *off = static_cast<long long>(z0) * plane;
        *n = static_cast<long long>(nz) * plane;
    };
    long long off = 0, n = 0;
    slab_of(me, &off, &n);
    if (me == 0) {
        if (dev_local)
            CUDA_CHECK(cudaMemcpyAsync(global_host + off, dev_local, sizeof(double) * n, cudaMemcpyDeviceToHost,
                                       ctx->stream));
        else
            std::memcpy(global_host + off, host_local, sizeof(double) * n);
        for (int r = 1; r < P; ++r) {
            long long ro = 0, rn = 0;
            slab_of(r, &ro, &rn);
            for (long long k = 0; k < rn; k += chunk) {
                const long long c = std::min(chunk, rn - k);
                if (stage.bytes < sizeof(double) * static_cast<size_t>(c)) stage.alloc(sizeof(double) * c, ctx->stream);
                NCCL_CHECK(ncclRecv(stage.p, static_cast<size_t>(c), ncclFloat64, r, ctx->comm, ctx->stream));
                CUDA_CHECK(cudaMemcpyAsync(global_host + ro + k, stage.p, sizeof(double) * c, cudaMemcpyDeviceToHost,
                                           ctx->stream));
                CUDA_CHECK(cudaStreamSynchronize(ctx->stream));
            }
        }
    } else {
        for (long long k = 0; k < n; k += chunk) {
            const long long c = std::min(chunk, n - k);
            const double* src = dev_local ? dev_local + k : nullptr;
            if (!dev_local) {
                if (stage.bytes < sizeof(double) * static_cast<size_t>(c)) stage.alloc(sizeof(double) * c, ctx->stream);
                CUDA_CHECK(cudaMemcpyAsync(stage.p, host_local + k, sizeof(double) * c, cudaMemcpyHostToDevice,
                                           ctx->stream));
                src = stage.as<double>();
            }
            NCCL_CHECK(ncclSend(src, static_cast<size_t>(c), ncclFloat64, 0, ctx->comm, ctx->stream));
            CUDA_CHECK(cudaStreamSynchronize(ctx->stream));
        }
    }
    CUDA_CHECK(cudaStreamSynchronize(ctx->stream));
    stage.release();
}

// One step with the field coming from and going back to host memory, the
// copies overlapped with the stage kernels (lsg_solver_step_host).  The input
// is uploaded in K chunks of planes along the last axis on a copy-in stream.
// After each chunk, every RK level computes every plane whose (2W+1)-plane
// stencil of the previous level is available (periodic wrap or clamped
// edge rule of the slab axis, as the kernels apply it), one launch per
// contiguous run.  Each run of finished planes goes back on a copy-out
// stream while later chunks are still arriving.  A plane's value is computed
// by the same kernels from the same inputs, so the result is bit-identical to
// upload + lsg_solver_step + download.  In-place RK updates are safe: level S
// writes plane z of the input buffer only after every reader of that plane
// (stage-1 stencils within W, the RK base at z) has run.
void step_host_pipelined(lsg_solver* s, double dt, const double* hin, double* hout, unsigned long long* range) {
    lsg_ctx* ctx = s->ctx;
    Slab& sl = s->slabs[0];
    const int nz = sl.nz, W = s->W;
    const long long plane = s->plane;
    const bool periodic = bc_of(&s->g, s->D - 1) == LSG_BC_PERIODIC;
    const int S = stages_of(s->method);
    // chunks of ~32 MiB (at least 4): the copy engines and the first level's
    // kernels overlap better with more, smaller chunks on large fields (512^3:
    // 32 chunks give 16.1 G end to end, 16 give 15.9 G, 4 gave 13.0 G), while
    // small fields keep 4 (101^3: 8.9 G with 4, 6.1 G with 16); every chunk
    // keeps >= 4W+2 planes
    const long long fbytes = static_cast<long long>(sizeof(double)) * sl.nodes;
    int K = static_cast<int>(std::max(4LL, std::min(48LL, fbytes >> 25)));
    K = std::max(2, std::min(K, nz / (4 * W + 2)));
    if (const char* e = std::getenv("LSG_PIPE_K")) K = std::max(2, std::min(64, std::atoi(e)));
    if (!s->cin) {
        CUDA_CHECK(cudaStreamCreateWithFlags(&s->cin, cudaStreamNonBlocking));
        CUDA_CHECK(cudaStreamCreateWithFlags(&s->cout, cudaStreamNonBlocking));
    }
    while (static_cast<int>(s->pipe_ev.size()) < 2) {
        cudaEvent_t e;
        CUDA_CHECK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        s->pipe_ev.push_back(e);
    }
    cudaEvent_t ev_start = s->pipe_ev[0], ev_done = s->pipe_ev[1];
    // level l reads u = ob[l-1], writes ob[l] (integrator.cpp:58-85 buffer use)
    const int a = s->cur;
    int ob[4] = {a, 0, 0, 0}, mode[4] = {0, MODE_EULER, MODE_COMBINE, MODE_COMBINE}, v0b[4] = {-1, -1, a, a};
    double cw[4] = {0.0, 0.0, 0.0, 0.0};
    if (s->method == LSG_CFL1) {
        ob[1] = 1 - a;
    } else if (s->method == LSG_CFL2) {
        ob[1] = 1 - a, ob[2] = a, cw[2] = 0.5;
    } else {
        ob[1] = (a + 1) % 3, ob[2] = (a + 2) % 3, ob[3] = a, cw[2] = 0.25, cw[3] = 2.0 / 3.0;
    }
    CUDA_CHECK(cudaEventRecord(ev_start, ctx->stream));  // earlier work on the buffers is done first
    CUDA_CHECK(cudaStreamWaitEvent(s->cin, ev_start, 0));
    // LSG_PIPE_TRACE=1: %globaltimer stamps after every upload chunk, compute
    // round and copy-out batch, printed relative to the step start (tuning aid)
    const bool trace = std::getenv("LSG_PIPE_TRACE") != nullptr;
    std::vector<std::string> tnames;
    unsigned long long* tbuf = nullptr;
    if (trace) CUDA_CHECK(cudaMallocAsync(&tbuf, 128 * sizeof(unsigned long long), ctx->stream));
    auto mark = [&](const std::string& what, cudaStream_t st) {
        if (!trace || tnames.size() >= 128) return;
        if (st != ctx->stream) {
            CUDA_CHECK(cudaEventRecord(ev_done, ctx->stream));  // tbuf allocated
            CUDA_CHECK(cudaStreamWaitEvent(st, ev_done, 0));
        }
        launch_stamp(tbuf + tnames.size(), st);
        tnames.push_back(what);
    };
    mark("start", s->cin);
    // upload plan: K chunks of planes in order (ranges in upload order).
    // Uploading a periodic axis's wrap planes first and tapering the last
    // chunk measured equal (512^3: 24.05 vs 24.01 ms per step; the copy-in
    // stream ends 0.8 ms before the step, so little is left to drain)
    std::vector<std::pair<int, int>> up;
    for (int j = 0; j < K; ++j)
        up.emplace_back(static_cast<int>(static_cast<long long>(nz) * j / K),
                        static_cast<int>(static_cast<long long>(nz) * (j + 1) / K));
    const int nup = static_cast<int>(up.size());
    while (static_cast<int>(s->pipe_ev.size()) < nup + 2) {
        cudaEvent_t e;
        CUDA_CHECK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        s->pipe_ev.push_back(e);
    }
    for (int j = 0; j < nup; ++j) {
        CUDA_CHECK(cudaMemcpyAsync(sl.f[a] + up[j].first * plane, hin + up[j].first * plane,
                                   sizeof(double) * static_cast<size_t>((up[j].second - up[j].first) * plane),
                                   cudaMemcpyHostToDevice, s->cin));
        CUDA_CHECK(cudaEventRecord(s->pipe_ev[2 + j], s->cin));
        mark("h2d chunk " + std::to_string(j), s->cin);
    }
    std::vector<std::vector<char>> done(S + 1, std::vector<char>(nz, 0));
    auto ready = [&](int l, int z) {
        for (int k = -W; k <= W; ++k) {
            int zz = z + k;
            if (periodic) zz = ((zz % nz) + nz) % nz;
            else zz = std::max(0, std::min(nz - 1, zz));
            if (!done[l - 1][zz]) return false;
        }
        return true;
    };
    // finished runs go back after every compute round, adjacent runs as one
    // copy (holding them back for larger copies measured slower: 512^3, 64 /
    // 128 / 256 MiB batches 25.9 / 26.6 / 28.3 ms per step against 24.2)
    std::vector<std::pair<int, int>> final_runs;
    for (int j = 0; j < nup; ++j) {
        for (int z = up[j].first; z < up[j].second; ++z) done[0][z] = 1;
        CUDA_CHECK(cudaStreamWaitEvent(ctx->stream, s->pipe_ev[2 + j], 0));
        for (int l = 1; l <= S; ++l) {
            for (int z = 0; z < nz;) {
                if (done[l][z] || !ready(l, z)) {
                    ++z;
                    continue;
                }
                int e = z;
                while (e < nz && !done[l][e] && ready(l, e)) ++e;
                launch_planes(s, sl, mode[l], ob[l - 1], v0b[l], ob[l], dt, cw[l], l == S ? range : nullptr, z, e, 0,
                              0, ctx->stream);
                for (int q = z; q < e; ++q) done[l][q] = 1;
                if (l == S) {
                    if (!final_runs.empty() && final_runs.back().second == z) final_runs.back().second = e;
                    else final_runs.emplace_back(z, e);
                }
                z = e;
            }
        }
        mark("compute round " + std::to_string(j), ctx->stream);
        if (!final_runs.empty()) {
            CUDA_CHECK(cudaEventRecord(ev_done, ctx->stream));
            CUDA_CHECK(cudaStreamWaitEvent(s->cout, ev_done, 0));
            for (const auto& r : final_runs)
                CUDA_CHECK(cudaMemcpyAsync(hout + r.first * plane, sl.f[ob[S]] + r.first * plane,
                                           sizeof(double) * static_cast<size_t>((r.second - r.first) * plane),
                                           cudaMemcpyDeviceToHost, s->cout));
            mark("d2h after round " + std::to_string(j), s->cout);
            final_runs.clear();
        }
    }
    for (int z = 0; z < nz; ++z)
        if (!done[S][z]) fail(LSG_ECUDA, "step_host: pipeline left planes unscheduled");
    CUDA_CHECK(cudaStreamSynchronize(s->cout));
    s->cur = ob[S];
    if (trace) {
        std::vector<unsigned long long> t(tnames.size());
        CUDA_CHECK(cudaDeviceSynchronize());
        CUDA_CHECK(cudaMemcpy(t.data(), tbuf, sizeof(unsigned long long) * t.size(), cudaMemcpyDeviceToHost));
        CUDA_CHECK(cudaFree(tbuf));
        for (size_t k = 0; k < t.size(); ++k)
            std::fprintf(stderr, "pipe %-22s %8.1f us\n", tnames[k].c_str(), 1e-3 * static_cast<double>(t[k] - t[0]));
    }
}

}  // namespace

// =============================== C ABI ======================================

extern "C" {

int lsg_abi_version(void) { return LSG_ABI_VERSION; }

const char* lsg_last_error(void) { return g_err.c_str(); }

void lsg_opts_default(lsg_opts* o) {
    if (o) *o = default_opts();
}

int lsg_device_count(int* count) {
    return guarded([&] {
        int n = 0;
        const cudaError_t e = cudaGetDeviceCount(&n);
        if (e != cudaSuccess) {
            cudaGetLastError();
            n = 0;
        }
        *count = n;
    });
}

int lsg_ctx_create(int device, lsg_ctx** out) {
    return guarded([&] {
        int n = 0;
        if (cudaGetDeviceCount(&n) != cudaSuccess || n == 0) {
            cudaGetLastError();
            fail(LSG_ECUDA, "no CUDA device is available (the B200 path has no CPU fallback)");
        }
        if (device < 0 || device >= n) fail(LSG_EINVAL, "device index out of range");
        auto c = std::make_unique<lsg_ctx>();
        c->device = device;
        CUDA_CHECK(cudaSetDevice(device));
        CUDA_CHECK(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
        *out = c.release();
    });
}

int lsg_nccl_unique_id(void* out128) {
    return guarded([&] {
        static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId size");
        ncclUniqueId id;
        NCCL_CHECK(ncclGetUniqueId(&id));
        std::memcpy(out128, &id, sizeof id);
    });
}

int lsg_ctx_create_dist(int device, int rank, int nranks, const void* nccl_id128, lsg_ctx** out) {
    return guarded([&] {
        if (nranks < 1 || rank < 0 || rank >= nranks) fail(LSG_EINVAL, "invalid rank/nranks");
        lsg_ctx* c = nullptr;
        const int rc = lsg_ctx_create(device, &c);
        if (rc) fail(rc, g_err);
        std::unique_ptr<lsg_ctx> owner(c);
        c->rank = rank;
        c->nranks = nranks;
        // LSG_DIST_SELFTEST=1 with nranks == 1: a real one-rank NCCL
        // communicator, and solvers take the distributed branch (halo planes,
        // NCCL self send/recv on a periodic slab axis, NCCL all-reduces), so
        // that branch runs on a one-GPU box without ranks waiting on each other.
        const char* st = std::getenv("LSG_DIST_SELFTEST");
        c->dist_selftest = nranks == 1 && st && std::string(st) == "1";
        if (nranks > 1 || c->dist_selftest) {
            ncclUniqueId id;
            std::memcpy(&id, nccl_id128, sizeof id);
            NCCL_CHECK(ncclCommInitRank(&c->comm, nranks, id, rank));
        }
        *out = owner.release();
    });
}

int lsg_ctx_destroy(lsg_ctx* ctx) {
    return guarded([&] {
        if (!ctx) return;
        cudaSetDevice(ctx->device);
        cudaStreamSynchronize(ctx->stream);
        delete ctx->cached;
        if (ctx->comm) ncclCommDestroy(ctx->comm);
        for (auto& b : ctx->scratch) b.release();
        cudaStreamDestroy(ctx->stream);
        delete ctx;
    });
}

int lsg_ctx_synchronize(lsg_ctx* ctx) {
    return guarded([&] {
        activate(ctx);
        CUDA_CHECK(cudaStreamSynchronize(ctx->stream));
    });
}

int lsg_ctx_launch_count(const lsg_ctx* ctx, uint64_t* count) {
    return guarded([&] {
        if (!ctx) fail(LSG_EINVAL, "null context");
        *count = ctx->launches;
    });
}

int lsg_host_alloc(size_t bytes, void** out) {
    return guarded([&] {
        *out = nullptr;
        CUDA_CHECK(cudaMallocHost(out, bytes));
    });
}

int lsg_host_free(void* p) {
    return guarded([&] {
        if (p) CUDA_CHECK(cudaFreeHost(p));
    });
}

int lsg_grid_check(const lsg_grid* g) {
    return guarded([&] { check_grid(g); });
}

int lsg_grid_spacing(const lsg_grid* g, int d, double* dx) {
    return guarded([&] {
        check_grid(g);
        if (d < 0 || d >= g->dim) fail(LSG_EINVAL, "grid: dimension out of range");
        *dx = spacing(g, d);
    });
}

int lsg_grid_node_count(const lsg_grid* g, size_t* n) {
    return guarded([&] {
        check_grid(g);
        *n = static_cast<size_t>(node_count(g));
    });
}

int lsg_grid_axis(const lsg_grid* g, int d, double* out) {
    return guarded([&] {
        check_grid(g);
        if (d < 0 || d >= g->dim) fail(LSG_EINVAL, "grid: dimension out of range");
        const double dx = spacing(g, d);
        for (int i = 0; i < g->counts[d]; ++i) out[i] = g->mins[d] + static_cast<double>(i) * dx;
    });
}

int lsg_halo_plan(int n, int nranks, int rank, int width, int periodic, int* kinds, int* peers, int* planes,
                  int* counts, int* n_messages) {
    return guarded([&] {
        if (n < 1 || nranks < 1 || rank < 0 || rank >= nranks || width < 0)
            fail(LSG_EINVAL, "halo_plan: invalid arguments");
        if (!kinds || !peers || !planes || !counts || !n_messages) fail(LSG_EINVAL, "halo_plan: null output");
        HaloMsg msg[4];
        const int k = halo_plan(n, nranks, rank, width, periodic != 0, msg);
        for (int i = 0; i < k; ++i) {
            kinds[i] = msg[i].kind;
            peers[i] = msg[i].peer;
            planes[i] = msg[i].plane;
            counts[i] = msg[i].count;
        }
        *n_messages = k;
    });
}

int lsg_slab_partition(int n, int nranks, int rank, int* z0, int* nz) {
    return guarded([&] {
        if (n < 1 || nranks < 1 || rank < 0 || rank >= nranks) fail(LSG_EINVAL, "slab_partition: invalid arguments");
        partition(n, nranks, rank, z0, nz);
    });
}

// ---- snapshot I/O (snapshot.cpp:69-129) -------------------------------------

int lsg_write_snapshot(const lsg_grid* g, const double* field, double time, const char* path) {
    return guarded([&] {
        check_grid(g);
        std::ofstream os(path, std::ios::binary);
        if (!os) fail(LSG_ENUMERIC, std::string("snapshot: cannot open ") + path + " for writing");
        std::ostringstream h;
        h.precision(17);
        h << "dims " << g->dim << "\n" << "counts";
        for (int d = 0; d < g->dim; ++d) h << " " << g->counts[d];
        h << "\nmins";
        for (int d = 0; d < g->dim; ++d) h << " " << g->mins[d];
        h << "\nmaxs";
        for (int d = 0; d < g->dim; ++d) h << " " << g->maxs[d];
        h << "\ntime " << time << "\n";
        os << h.str();
        static_assert(sizeof(double) == 8, "fp64");
        os.write(reinterpret_cast<const char*>(field), static_cast<std::streamsize>(sizeof(double) * node_count(g)));
        if (!os) fail(LSG_ENUMERIC, std::string("snapshot: write to ") + path + " failed");
    });
}

int lsg_read_snapshot(const char* path, lsg_grid* g, double* time, double* field, size_t cap) {
    return guarded([&] {
        std::ifstream is(path, std::ios::binary);
        if (!is) fail(LSG_ENUMERIC, std::string("snapshot: cannot open ") + path);
        auto line = [&](const std::string& key) {
            std::string l;
            if (!std::getline(is, l)) fail(LSG_ENUMERIC, "snapshot: truncated header, expected '" + key + "'");
            if (l.rfind(key + " ", 0) != 0 && l != key)
                fail(LSG_ENUMERIC, "snapshot: expected header line '" + key + "', got '" + l + "'");
            return l.size() > key.size() ? l.substr(key.size() + 1) : std::string();
        };
        const int dims = std::stoi(line("dims"));
        if (dims < 1 || dims > 16) fail(LSG_ENUMERIC, "snapshot: implausible dimension count");
        if (dims > LSG_MAX_DIM) fail(LSG_EINVAL, "snapshot: the device path supports at most 6 dimensions");
        lsg_grid out{};
        out.dim = dims;
        auto reals = [&](const std::string& key, double* dst, int n) {
            std::istringstream ss(line(key));
            int k = 0;
            double v;
            while (ss >> v) {
                if (k < n) dst[k] = v;
                ++k;
            }
            if (k != n) fail(LSG_ENUMERIC, "snapshot: header line '" + key + "' has wrong arity");
        };
        {
            std::istringstream cs(line("counts"));
            int k = 0, c;
            while (cs >> c) {
                if (k < dims) out.counts[k] = c;
                ++k;
            }
            if (k != dims) fail(LSG_ENUMERIC, "snapshot: header line 'counts' has wrong arity");
        }
        reals("mins", out.mins, dims);
        reals("maxs", out.maxs, dims);
        double t = 0.0;
        reals("time", &t, 1);
        check_grid(&out);
        *g = out;
        if (time) *time = t;
        if (field) {
            const long long N = node_count(&out);
            if (static_cast<long long>(cap) < N) fail(LSG_EINVAL, "snapshot: output buffer too small");
            is.read(reinterpret_cast<char*>(field), static_cast<std::streamsize>(sizeof(double) * N));
            if (!is) fail(LSG_ENUMERIC, std::string("snapshot: payload truncated in ") + path);
            for (long long i = 0; i < N; ++i)
                if (!std::isfinite(field[i])) fail(LSG_ENUMERIC, "snapshot: payload contains non-finite values");
        }
    });
}

int lsg_extract_zero_set_2d(lsg_ctx* ctx, const lsg_grid* g, const double* field, double* segments, size_t cap,
                            size_t* n_segments) {
    return guarded([&] {
        activate(ctx);
        check_grid(g);
        if (g->dim != 2) fail(LSG_EINVAL, "extract_zero_set_2d: field must be 2-D");  // contour.cpp:29-30
        const int nx = g->counts[0], ny = g->counts[1];
        const long long N = node_count(g);
        const int ncells = (nx - 1) * (ny - 1);
        double* df = ctx->staging(0, sizeof(double) * N);
        std::vector<double> axes(static_cast<size_t>(nx + ny));
        for (int i = 0; i < nx; ++i) axes[i] = g->mins[0] + static_cast<double>(i) * spacing(g, 0);
        for (int j = 0; j < ny; ++j) axes[nx + j] = g->mins[1] + static_cast<double>(j) * spacing(g, 1);
        double* dax = ctx->staging(1, sizeof(double) * axes.size());
        const size_t tb = zero_set_temp_bytes(ncells);
        // counts | offsets | cub temp in one staging buffer
        const size_t ib = (sizeof(int) * static_cast<size_t>(ncells) + 255) & ~size_t(255);
        char* scratch = reinterpret_cast<char*>(ctx->staging(2, 2 * ib + tb + 256));
        CUDA_CHECK(cudaMemcpyAsync(df, field, sizeof(double) * N, cudaMemcpyHostToDevice, ctx->stream));
        CUDA_CHECK(cudaMemcpyAsync(dax, axes.data(), sizeof(double) * axes.size(), cudaMemcpyHostToDevice, ctx->stream));
        const long long cap_dev = static_cast<long long>(cap);
        double* dseg = cap ? ctx->staging(3, sizeof(double) * 4 * cap) : nullptr;
        int total = 0;
        zero_set_2d(df, nx, ny, dax, dax + nx, spacing(g, 0), spacing(g, 1), dseg, cap_dev,
                    reinterpret_cast<int*>(scratch), reinterpret_cast<int*>(scratch + ib), scratch + 2 * ib, tb,
                    ctx->stream, &total);
        ctx->note_launch(3);
        if (n_segments) *n_segments = static_cast<size_t>(total);
        if (static_cast<size_t>(total) > cap) fail(LSG_ERANGE, "extract_zero_set_2d: segment buffer too small");
        if (total)
            CUDA_CHECK(cudaMemcpyAsync(segments, dseg, sizeof(double) * 4 * total, cudaMemcpyDeviceToHost, ctx->stream));
        CUDA_CHECK(cudaStreamSynchronize(ctx->stream));
    });
}

int lsg_slice_2d(lsg_ctx* ctx, const lsg_grid* g, const double* field, int fixed_dim, int index, double* out) {
    return guarded([&] {
        activate(ctx);
        check_grid(g);
        // contour.cpp:101-106
        if (g->dim < 3) fail(LSG_EINVAL, "slice_2d: field must be at least 3-D");
        if (fixed_dim < 0 || fixed_dim >= g->dim) fail(LSG_EINVAL, "slice_2d: fixed dimension out of range");
        if (index < 0 || index >= g->counts[fixed_dim]) fail(LSG_EINVAL, "slice_2d: slice index out of range");
        if (g->dim != 3) fail(LSG_EINVAL, "slice_2d: the device path slices 3-D fields");
        long long st[LSG_MAX_DIM], acc = 1;
        for (int d = 0; d < g->dim; ++d) st[d] = acc, acc *= g->counts[d];
        int kept[2], k = 0;
        for (int d = 0; d < 3; ++d)
            if (d != fixed_dim) kept[k++] = d;
        const long long N = node_count(g);
        const long long total = static_cast<long long>(g->counts[kept[0]]) * g->counts[kept[1]];
        double* df = ctx->staging(0, sizeof(double) * N);
        double* dout = ctx->staging(1, sizeof(double) * total);
        CUDA_CHECK(cudaMemcpyAsync(df, field, sizeof(double) * N, cudaMemcpyHostToDevice, ctx->stream));
        launch_slice(df, total, g->counts[kept[0]], st[kept[0]], st[kept[1]], index * st[fixed_dim], dout, ctx->stream);
        ctx->note_launch();
        CUDA_CHECK(cudaMemcpyAsync(out, dout, sizeof(double) * total, cudaMemcpyDeviceToHost, ctx->stream));
        CUDA_CHECK(cudaStreamSynchronize(ctx->stream));
    });
}

int lsg_pad_ghost(lsg_ctx* ctx, const lsg_grid* g, const double* field, int dim, int width, double* out) {
    return guarded([&] {
        activate(ctx);
        check_grid(g);
        if (dim < 0 || dim >= g->dim) fail(LSG_EINVAL, "pad_ghost: dimension out of range");
        if (width < 1) fail(LSG_EINVAL, "pad_ghost: width must be >= 1");
        const int n = g->counts[dim];
        if (width >= n) fail(LSG_EINVAL, "pad_ghost: width must be smaller than the node count along dim");
        const long long N = node_count(g);
        const long long n_out = N / n * (n + 2 * width);
        long long stride = 1;
        for (int d = 0; d < dim; ++d) stride *= g->counts[d];
        double* du = ctx->staging(0, sizeof(double) * N);
        double* dout = ctx->staging(1, sizeof(double) * n_out);
        CUDA_CHECK(cudaMemcpyAsync(du, field, sizeof(double) * N, cudaMemcpyHostToDevice, ctx->stream));
        launch_pad(du, dout, n_out, n, stride, width, bc_of(g, dim), ctx->stream);
        ctx->note_launch();
        CUDA_CHECK(cudaMemcpyAsync(out, dout, sizeof(double) * n_out, cudaMemcpyDeviceToHost, ctx->stream));
        CUDA_CHECK(cudaStreamSynchronize(ctx->stream));
    });
}

int lsg_shift_along_dim(lsg_ctx* ctx, const lsg_grid* g, const double* padded, int dim, int width, int offset,
                        double* out) {
    return guarded([&] {
        activate(ctx);
        check_grid(g);
        if (dim < 0 || dim >= g->dim) fail(LSG_EINVAL, "shift_along_dim: dimension out of range");
        if (width < 0) fail(LSG_EINVAL, "shift_along_dim: width must be >= 0");
        if (offset < -width || offset > width)
            fail(LSG_EINVAL, "shift_along_dim: |offset| must not exceed the ghost width");
        const int n = g->counts[dim];
        const long long N = node_count(g);
        const long long n_in = N / n * (n + 2 * width);
        long long stride = 1;
        for (int d = 0; d < dim; ++d) stride *= g->counts[d];
        double* din = ctx->staging(0, sizeof(double) * n_in);
        double* dout = ctx->staging(1, sizeof(double) * N);
        CUDA_CHECK(cudaMemcpyAsync(din, padded, sizeof(double) * n_in, cudaMemcpyHostToDevice, ctx->stream));
        launch_shift(din, dout, N, n, stride, width, offset, ctx->stream);
        ctx->note_launch();
        CUDA_CHECK(cudaMemcpyAsync(out, dout, sizeof(double) * N, cudaMemcpyDeviceToHost, ctx->stream));
        CUDA_CHECK(cudaStreamSynchronize(ctx->stream));
    });
}

int lsg_upwind(lsg_ctx* ctx, const lsg_grid* g, const double* v, int dim, int scheme, double* left, double* right) {
    return guarded([&] {
        activate(ctx);
        check_grid(g);
        if (scheme < LSG_SCHEME_FIRST || scheme > LSG_SCHEME_WENO5) fail(LSG_EINVAL, "unknown derivative scheme");
        const char* name = scheme_name(scheme);
        if (dim < 0 || dim >= g->dim) fail(LSG_EINVAL, std::string(name) + ": dimension out of range");
        if (g->counts[dim] < min_nodes(scheme))
            fail(LSG_EINVAL, std::string(name) + ": needs at least " + std::to_string(min_nodes(scheme)) +
                                 " nodes along dim " + std::to_string(dim));
        const long long N = node_count(g);
        double* du = ctx->staging(0, sizeof(double) * N);
        double* dl = ctx->staging(1, sizeof(double) * N);
        double* dr = ctx->staging(2, sizeof(double) * N);
        CUDA_CHECK(cudaMemcpyAsync(du, v, sizeof(double) * N, cudaMemcpyHostToDevice, ctx->stream));
        StageParams P{};
        P.u = du;
        P.n_local = N;
        long long st = 1;
        for (int d = 0; d < g->dim; ++d) {
            P.n[d] = g->counts[d];
            P.stride[d] = st;
            st *= g->counts[d];
            P.bc[d] = bc_of(g, d);
            P.lc[d] = line_const(g, d);
        }
        launch_upwind(P, dim, g->dim, scheme, dl, dr, ctx->stream);
        ctx->note_launch();
        CUDA_CHECK(cudaMemcpyAsync(left, dl, sizeof(double) * N, cudaMemcpyDeviceToHost, ctx->stream));
        CUDA_CHECK(cudaMemcpyAsync(right, dr, sizeof(double) * N, cudaMemcpyDeviceToHost, ctx->stream));
        CUDA_CHECK(cudaStreamSynchronize(ctx->stream));
    });
}

int lsg_term_lf(lsg_ctx* ctx, const lsg_grid* g, const lsg_problem* p, double t, const double* v, double* dvdt,
                double* step_bound) {
    (void)t;
    return guarded([&] {
        lsg_solver* s = cached_solver(ctx, g, p, LSG_CFL1);
        CallCache call_cache{ctx};
        if (!s->invalid.empty()) fail(LSG_EINVAL, s->invalid);
        upload(s, v, 0);
        ensure_alpha(s);
        CUDA_CHECK(cudaMemsetAsync(s->dflags.p, 0, sizeof(unsigned), ctx->stream));
        run_stage(s, MODE_TERM, 0, -1, 1, 0.0, 0.0, nullptr);  // halo exchange first on a multi-rank context
        if (s->distributed) {  // every rank raises the same error
            join_comm(s);
            NCCL_CHECK(ncclAllReduce(s->dflags.p, s->dflags.p, 1, ncclUint32, ncclMax, ctx->comm, ctx->stream));
        }
        unsigned flags = 0;
        CUDA_CHECK(cudaMemcpyAsync(&flags, s->dflags.p, sizeof flags, cudaMemcpyDeviceToHost, ctx->stream));
        CUDA_CHECK(cudaStreamSynchronize(ctx->stream));
        // hamiltonian.cpp:37-56: H is validated before the bounds
        if (flags & FLAG_HAM_NONFINITE)
            fail(LSG_ENUMERIC, "term_lax_friedrichs: hamiltonian produced a non-finite value");
        check_alpha_valid(s);
        download(s, dvdt, 1);
        *step_bound = s->bound;
    });
}

// The device Hamiltonian (dim < 0) or the dissipation bound of one dimension
// on host fields: the reference's plugins (HamiltonianFn / DissipationFn,
// hamiltonian.hpp:16-25) for the device kinds.
void eval_plugin(lsg_ctx* ctx, const lsg_grid* g, const lsg_problem* p, const double* const* costate, int dim,
                 double* out) {
    lsg_solver* s = cached_solver(ctx, g, p, LSG_CFL1);
    CallCache call_cache{ctx};
    if (s->slabs.size() != 1 || s->distributed) fail(LSG_EINVAL, "plugin evaluation needs a single-rank context");
    EvalFn fn = lookup_eval(p->kind, g->dim);
    if (!fn) fail(LSG_EINVAL, "hamiltonian: kind not available for this grid dimension");
    if (dim >= g->dim) fail(LSG_EINVAL, "dissipation: dimension out of range");
    const long long N = s->total;
    EvalParams E{};
    E.P = slab_params(s, s->slabs[0]);
    E.dim = dim;
    if (dim < 0) {
        double* dc = ctx->staging(0, sizeof(double) * static_cast<size_t>(N * g->dim));
        for (int d = 0; d < g->dim; ++d) {
            if (!costate || !costate[d]) fail(LSG_EINVAL, "hamiltonian: costate must hold one field per dimension");
            CUDA_CHECK(cudaMemcpyAsync(dc + d * N, costate[d], sizeof(double) * N, cudaMemcpyHostToDevice,
                                       ctx->stream));
            E.costate[d] = dc + d * N;
        }
    }
    double* dout = ctx->staging(1, sizeof(double) * static_cast<size_t>(N));
    E.out = dout;
    void* args[] = {&E};
    CUDA_CHECK(cudaLaunchKernel(reinterpret_cast<const void*>(fn), dim3(static_cast<unsigned>((N + 255) / 256)),
                                dim3(256), args, 0, ctx->stream));
    ctx->note_launch();
    CUDA_CHECK(cudaMemcpyAsync(out, dout, sizeof(double) * N, cudaMemcpyDeviceToHost, ctx->stream));
    CUDA_CHECK(cudaStreamSynchronize(ctx->stream));
}

int lsg_eval_hamiltonian(lsg_ctx* ctx, const lsg_grid* g, const lsg_problem* p, double t,
                         const double* const* costate, double* out) {
    (void)t;  // every device kind is time-invariant
    return guarded([&] {
        if (!out) fail(LSG_EINVAL, "hamiltonian: null output");
        eval_plugin(ctx, g, p, costate, -1, out);
    });
}

int lsg_eval_dissipation(lsg_ctx* ctx, const lsg_grid* g, const lsg_problem* p, double t, int dim, double* out) {
    (void)t;
    return guarded([&] {
        if (!out) fail(LSG_EINVAL, "dissipation: null output");
        if (dim < 0) fail(LSG_EINVAL, "dissipation: dimension out of range");
        eval_plugin(ctx, g, p, nullptr, dim, out);
    });
}

int lsg_set_op(lsg_ctx* ctx, int op, size_t n, const double* a, const double* b, double* out) {
    return guarded([&] {
        activate(ctx);
        if (op < 1 || op > 3) fail(LSG_EINVAL, "set_op: unknown operation");
        if (n == 0) return;
        if (!a || !out || (op != 3 && !b)) fail(LSG_EINVAL, "set_op: null buffer");
        double* da = ctx->staging(0, sizeof(double) * n);
        double* db = ctx->staging(1, sizeof(double) * n);
        double* dout = ctx->staging(2, sizeof(double) * n);
        CUDA_CHECK(cudaMemcpyAsync(da, a, sizeof(double) * n, cudaMemcpyHostToDevice, ctx->stream));
        if (op != 3) CUDA_CHECK(cudaMemcpyAsync(db, b, sizeof(double) * n, cudaMemcpyHostToDevice, ctx->stream));
        launch_set_op(op, static_cast<long long>(n), da, db, dout, ctx->stream);
        ctx->note_launch();
        CUDA_CHECK(cudaMemcpyAsync(out, dout, sizeof(double) * n, cudaMemcpyDeviceToHost, ctx->stream));
        CUDA_CHECK(cudaStreamSynchronize(ctx->stream));
    });
}

int lsg_restrict_update(lsg_ctx* ctx, size_t n, const double* dvdt, int direction, double* out) {
    return guarded([&] {
        activate(ctx);
        if (n == 0) return;
        double* din = ctx->staging(0, sizeof(double) * n);
        double* dout = ctx->staging(1, sizeof(double) * n);
        CUDA_CHECK(cudaMemcpyAsync(din, dvdt, sizeof(double) * n, cudaMemcpyHostToDevice, ctx->stream));
        launch_restrict(din, dout, static_cast<long long>(n), direction, ctx->stream);
        ctx->note_launch();
        CUDA_CHECK(cudaMemcpyAsync(out, dout, sizeof(double) * n, cudaMemcpyDeviceToHost, ctx->stream));
        CUDA_CHECK(cudaStreamSynchronize(ctx->stream));
    });
}

int lsg_integrate(lsg_ctx* ctx, const lsg_grid* g, const lsg_problem* p, int method, double t0, double tf, double* v,
                  const lsg_opts* opts, lsg_steplog* steps, size_t log_cap, size_t* n_steps, double* t_final) {
    return guarded([&] {
        if (opts) check_options(opts);
        lsg_solver* s = cached_solver(ctx, g, p, method);
        CallCache call_cache{ctx};
        LegPlan plan = plan_leg(s, t0, tf, opts);
        check_log_room(plan.log.size(), steps, log_cap, n_steps);
        upload(s, v, 0);
        run_leg(s, plan);
        download(s, v, s->cur);
        copy_log(plan.log, steps, log_cap, n_steps);
        if (t_final) *t_final = plan.t_final;
    });
}

}  // extern "C"

namespace {

// solve_brt (reachability.cpp:135-174) from checkpoint k_start: the field
// v_start at integration time t_start; legs k_start+1 .. n_checkpoints-1 run
// as the reference's (equal durations from 0, each leg starting where the
// previous one stopped), checkpoints[0] = v_start.  k_start = 0, t_start = 0
// is the reference's solve_brt; k_start > 0 resumes a checkpointed run (the
// reference has no resume).
void solve_brt_from(lsg_ctx* ctx, const lsg_grid* g, const lsg_problem* p, const double* v_start, int k_start,
                    double t_start, double t_first, double t_second, int n_checkpoints, int method,
                    const lsg_opts* opts, double* checkpoints, double* checkpoint_times, int* n_out,
                    lsg_steplog* steps, size_t log_cap, size_t* n_steps, double* integration_seconds) {
    activate(ctx);
    check_grid(g);
    // reachability.cpp:138-143
    if (n_checkpoints < 1) fail(LSG_EINVAL, "solve_brt: need at least one checkpoint");
    if (!std::isfinite(t_first) || !std::isfinite(t_second)) fail(LSG_EINVAL, "solve_brt: tspan must be finite");
    if (k_start < 0 || k_start >= n_checkpoints) fail(LSG_EINVAL, "solve_brt: resume checkpoint out of range");
    if (!std::isfinite(t_start)) fail(LSG_EINVAL, "solve_brt: resume time must be finite");
    long long N = node_count(g);
    if (ctx->nranks > 1) {  // distributed context: v0 and the checkpoints are this rank's slab
        int z0 = 0, nz = 0;
        partition(g->counts[g->dim - 1], ctx->nranks, ctx->rank, &z0, &nz);
        N = N / g->counts[g->dim - 1] * nz;
    }
    const double duration = std::abs(t_second - t_first);
    const int segments = n_checkpoints - 1;
    std::memcpy(checkpoints, v_start, sizeof(double) * N);
    checkpoint_times[0] = k_start == 0 ? 0.0
                                       : duration * static_cast<double>(k_start) / static_cast<double>(segments);
    *n_out = 1;
    if (n_steps) *n_steps = 0;
    if (integration_seconds) *integration_seconds = 0.0;
    if (duration == 0.0 || n_checkpoints == 1 || k_start == segments) return;
    lsg_solver* s = cached_solver(ctx, g, p, method);
    CallCache call_cache{ctx};
    // every leg's schedule up front (reachability.cpp:160-170: the next leg
    // starts from leg.t), so the log capacity is known before device work
    std::vector<LegPlan> plans;
    size_t total = 0;
    double t = t_start;
    for (int k = k_start + 1; k <= segments; ++k) {
        const double t_end = duration * static_cast<double>(k) / static_cast<double>(segments);
        plans.push_back(plan_leg(s, t, t_end, opts));
        t = plans.back().t_final;
        total += plans.back().log.size();
        if (plans.back().collapsed || plans.back().bound_invalid) break;
    }
    check_log_room(total, steps, log_cap, n_steps);
    upload(s, v_start, 0);
    std::vector<lsg_steplog> all;
    const auto start = std::chrono::steady_clock::now();
    for (int i = 0; i < static_cast<int>(plans.size()); ++i) {
        const int k = k_start + 1 + i;
        const double t_end = duration * static_cast<double>(k) / static_cast<double>(segments);
        run_leg(s, plans[i]);
        all.insert(all.end(), plans[i].log.begin(), plans[i].log.end());
        download(s, checkpoints + static_cast<long long>(i + 1) * N, s->cur);
        checkpoint_times[i + 1] = t_end;
        *n_out = i + 2;
    }
    const auto stop = std::chrono::steady_clock::now();
    if (integration_seconds) *integration_seconds = std::chrono::duration<double>(stop - start).count();
    copy_log(all, steps, log_cap, n_steps);
}

}  // namespace

extern "C" {

int lsg_solve_brt(lsg_ctx* ctx, const lsg_grid* g, const lsg_problem* p, const double* v0, double t_first,
                  double t_second, int n_checkpoints, int method, const lsg_opts* opts, double* checkpoints,
                  double* checkpoint_times, int* n_out, lsg_steplog* steps, size_t log_cap, size_t* n_steps,
                  double* integration_seconds) {
    return guarded([&] {
        solve_brt_from(ctx, g, p, v0, 0, 0.0, t_first, t_second, n_checkpoints, method, opts, checkpoints,
                       checkpoint_times, n_out, steps, log_cap, n_steps, integration_seconds);
    });
}

int lsg_solve_brt_resume(lsg_ctx* ctx, const lsg_grid* g, const lsg_problem* p, const double* v_k, int k,
                         double t_k, double t_first, double t_second, int n_checkpoints, int method,
                         const lsg_opts* opts, double* checkpoints, double* checkpoint_times, int* n_out,
                         lsg_steplog* steps, size_t log_cap, size_t* n_steps, double* integration_seconds) {
    return guarded([&] {
        solve_brt_from(ctx, g, p, v_k, k, t_k, t_first, t_second, n_checkpoints, method, opts, checkpoints,
                       checkpoint_times, n_out, steps, log_cap, n_steps, integration_seconds);
    });
}

// ---- device-resident solver ----------------------------------------------

int lsg_solver_create(lsg_ctx* ctx, const lsg_grid* global_grid, const lsg_problem* p, int method,
                      lsg_solver** out) {
    return guarded([&] { *out = make_solver_retry(ctx, global_grid, p, method, 1).release(); });
}

int lsg_solver_create_slabs(lsg_ctx* ctx, const lsg_grid* global_grid, const lsg_problem* p, int method, int nslabs,
                            lsg_solver** out) {
    return guarded([&] {
        if (!ctx) fail(LSG_EINVAL, "null context");
        if (ctx->nranks > 1) fail(LSG_EINVAL, "in-process slabs need a single-rank context");
        if (nslabs < 1) fail(LSG_EINVAL, "nslabs must be >= 1");
        *out = make_solver_retry(ctx, global_grid, p, method, nslabs).release();
    });
}

int lsg_solver_destroy(lsg_solver* s) {
    return guarded([&] {
        if (!s) return;
        cudaSetDevice(s->ctx->device);
        // work a caller queued on lsg_solver_field_device's pointer from its own
        // streams must finish before the memory is recycled
        cudaDeviceSynchronize();
        delete s;
    });
}

int lsg_solver_slab(const lsg_solver* s, int* z0, int* nz, size_t* local_nodes) {
    return guarded([&] {
        if (!s) fail(LSG_EINVAL, "null solver");
        if (s->distributed) {
            *z0 = s->slabs[0].z0;
            *nz = s->slabs[0].nz;
            *local_nodes = static_cast<size_t>(s->slabs[0].nodes);
        } else {
            *z0 = 0;
            *nz = s->g.counts[s->D - 1];
            *local_nodes = static_cast<size_t>(s->total);
        }
    });
}

int lsg_solver_set_field(lsg_solver* s, const double* host_v) {
    return guarded([&] {
        if (!s) fail(LSG_EINVAL, "null solver");
        if (!host_v) fail(LSG_EINVAL, "set_field: null host buffer");
        activate(s->ctx);
        s->cur = 0;
        upload(s, host_v, 0);
        CUDA_CHECK(cudaStreamSynchronize(s->ctx->stream));
    });
}

int lsg_solver_get_field(lsg_solver* s, double* host_v) {
    return guarded([&] {
        if (!s) fail(LSG_EINVAL, "null solver");
        if (!host_v) fail(LSG_EINVAL, "get_field: null host buffer");
        activate(s->ctx);
        download(s, host_v, s->cur);
    });
}

int lsg_solver_set_field_device(lsg_solver* s, const double* dev_v) {
    return guarded([&] {
        if (!s) fail(LSG_EINVAL, "null solver");
        if (!dev_v) fail(LSG_EINVAL, "set_field_device: null device pointer");
        activate(s->ctx);
        s->cur = 0;
        invalidate_halos(s);
        for (const Slab& sl : s->slabs) {
            const long long off = s->distributed ? 0 : static_cast<long long>(sl.z0) * s->plane;
            CUDA_CHECK(cudaMemcpyAsync(sl.f[0], dev_v + off, sizeof(double) * sl.nodes, cudaMemcpyDeviceToDevice,
                                       s->ctx->stream));
        }
    });
}

int lsg_solver_field_device(lsg_solver* s, double** dev_v) {
    return guarded([&] {
        if (!s) fail(LSG_EINVAL, "null solver");
        if (!dev_v) fail(LSG_EINVAL, "field_device: null output");
        if (s->slabs.size() != 1) fail(LSG_EINVAL, "field_device: solver holds several slabs");
        *dev_v = s->slabs[0].f[s->cur];
        invalidate_halos(s);  // the caller may write through the pointer
    });
}

int lsg_solver_apply_shape(lsg_solver* s, int op, int shape, unsigned ignored_mask, const double* center,
                           const double* upper, double radius) {
    return guarded([&] {
        if (!s) fail(LSG_EINVAL, "null solver");
        activate(s->ctx);
        if (op < 0 || op > 2) fail(LSG_EINVAL, "apply_shape: unknown operation");
        if (shape < 0 || shape > 4) fail(LSG_EINVAL, "init_shape: unknown shape");
        // implicit_surfaces.cpp argument checks, same messages
        if (shape <= 2 && !(radius > 0.0)) fail(LSG_EINVAL, "init_shape: radius must be positive");
        if (shape == 2 && s->D != 6) fail(LSG_EINVAL, "init_shape: pair distance needs a 6-D grid");
        if (shape == 1) {
            if (ignored_mask == 0) fail(LSG_EINVAL, "cylinder: ignored_dims must be nonempty");
            if (ignored_mask >> s->D) fail(LSG_EINVAL, "cylinder: ignored dimension out of range");
            if (__builtin_popcount(ignored_mask) >= s->D)
                fail(LSG_EINVAL, "cylinder: at least one dimension must remain active");
        }
        if (shape == 3) {
            if (!center || !upper) fail(LSG_EINVAL, "rectangle: corner length must equal the grid dimension");
            for (int d = 0; d < s->D; ++d)
                if (!(upper[d] > center[d]))
                    fail(LSG_EINVAL, "rectangle: upper must exceed lower in dimension " + std::to_string(d));
        }
        if (shape == 4) {
            if (s->D != 2 && s->D != 3) fail(LSG_EINVAL, "ellipsoid: only 2-D and 3-D grids are supported");
            if (!(radius > 0.0)) fail(LSG_EINVAL, "ellipsoid: radius must be positive");
        }
        if (op == 0) s->cur = 0;  // a fresh field; compositions act on the current one
        invalidate_halos(s);
        for (Slab& sl : s->slabs) {
            ShapeParams S{};
            S.n_local = sl.nodes;
            S.D = s->D;
            for (int d = 0; d < s->D; ++d) {
                S.n[d] = d == s->D - 1 ? sl.nz : s->g.counts[d];
                S.axis[d] = s->axis[d];
                S.center[d] = center ? center[d] : 0.0;
                S.upper[d] = upper ? upper[d] : 0.0;
            }
            S.z0 = sl.z0;
            S.shape = shape;
            S.op = op;
            S.ignored_mask = shape == 1 ? ignored_mask : 0u;
            S.radius = radius;
            S.out = sl.f[s->cur];
            launch_shape(S, s->ctx->stream);
            s->ctx->note_launch();
        }
    });
}

int lsg_solver_init_shape(lsg_solver* s, int shape, unsigned ignored_mask, const double* center, double radius) {
    if (shape > 2) return guarded([&] { fail(LSG_EINVAL, "init_shape: unknown shape"); });
    return lsg_solver_apply_shape(s, 0, shape, ignored_mask, center, nullptr, radius);
}

int lsg_solver_complement(lsg_solver* s) {
    return guarded([&] {
        if (!s) fail(LSG_EINVAL, "null solver");
        activate(s->ctx);
        invalidate_halos(s);
        for (Slab& sl : s->slabs) {
            launch_set_op(3, sl.nodes, sl.f[s->cur], sl.f[s->cur], sl.f[s->cur], s->ctx->stream);
            s->ctx->note_launch();
        }
    });
}

int lsg_solver_step_bound(lsg_solver* s, double t, double* bound) {
    (void)t;
    return guarded([&] {
        if (!s) fail(LSG_EINVAL, "null solver");
        if (!bound) fail(LSG_EINVAL, "step_bound: null output");
        activate(s->ctx);
        check_alpha_valid(s);
        *bound = s->bound;
    });
}

int lsg_solver_step(lsg_solver* s, double t, double dt) {
    (void)t;
    return guarded([&] {
        if (!s) fail(LSG_EINVAL, "null solver");
        activate(s->ctx);
        check_alpha_valid(s);
        if (s->ring_next >= s->range_cap) ensure_range(s, s->range_cap);
        enqueue_step(s, dt, s->drange.as<unsigned long long>() + kRangeWords * s->ring_next);
        ++s->ring_next;
    });
}

int lsg_solver_step_host(lsg_solver* s, double t, double dt, const double* host_in, double* host_out) {
    (void)t;
    return guarded([&] {
        if (!s) fail(LSG_EINVAL, "null solver");
        if (!host_in || !host_out) fail(LSG_EINVAL, "step_host: null host buffer");
        activate(s->ctx);
        check_alpha_valid(s);
        if (s->ring_next >= s->range_cap) ensure_range(s, s->range_cap);
        unsigned long long* range = s->drange.as<unsigned long long>() + kRangeWords * s->ring_next;
        ++s->ring_next;
        const char* e = std::getenv("LSG_PIPE");
        const bool pipe = !(e && std::string(e) == "0");
        if (pipe && s->slabs.size() == 1 && !s->distributed && s->halo_w == 0 && s->slabs[0].nz >= 2 * (4 * s->W + 2)) {
            invalidate_halos(s);
            step_host_pipelined(s, dt, host_in, host_out, range);
        } else {  // several slabs or ranks, or too few planes to pipeline
            upload(s, host_in, s->cur);
            enqueue_step(s, dt, range);
            download(s, host_out, s->cur);
        }
    });
}

int lsg_solver_step_timed(lsg_solver* s, double t, double dt, double* stage_ms, double* step_ms) {
    (void)t;
    return guarded([&] {
        if (!s) fail(LSG_EINVAL, "null solver");
        if (!stage_ms || !step_ms) fail(LSG_EINVAL, "step_timed: null output");
        activate(s->ctx);
        check_alpha_valid(s);
        if (s->ring_next >= s->range_cap) ensure_range(s, s->range_cap);
        const int n = stages_of(s->method);
        cudaEvent_t ev[4];
        for (int k = 0; k <= n; ++k) CUDA_CHECK(cudaEventCreate(&ev[k]));
        enqueue_step(s, dt, s->drange.as<unsigned long long>() + kRangeWords * s->ring_next, ev);
        ++s->ring_next;
        CUDA_CHECK(cudaEventSynchronize(ev[n]));
        for (int k = 0; k < n; ++k) {
            float ms = 0.f;
            CUDA_CHECK(cudaEventElapsedTime(&ms, ev[k], ev[k + 1]));
            stage_ms[k] = ms;
        }
        float total = 0.f;
        CUDA_CHECK(cudaEventElapsedTime(&total, ev[0], ev[n]));
        *step_ms = total;
        for (int k = 0; k <= n; ++k) cudaEventDestroy(ev[k]);
    });
}

int lsg_solver_integrate(lsg_solver* s, double t0, double tf, const lsg_opts* opts, lsg_steplog* steps,
                         size_t log_cap, size_t* n_steps, double* t_final) {
    return guarded([&] {
        if (!s) fail(LSG_EINVAL, "null solver");
        activate(s->ctx);
        LegPlan plan = plan_leg(s, t0, tf, opts);
        check_log_room(plan.log.size(), steps, log_cap, n_steps);
        run_leg(s, plan);
        copy_log(plan.log, steps, log_cap, n_steps);
        if (t_final) *t_final = plan.t_final;
    });
}

int lsg_solver_write_snapshot(lsg_solver* s, double time, const char* path) {
    return guarded([&] {
        if (!s) fail(LSG_EINVAL, "null solver");
        activate(s->ctx);
        const size_t n = static_cast<size_t>(s->total);
        if (s->distributed) {  // collective: the slabs gathered on rank 0, which writes the whole grid
            if (s->ctx->rank == 0 && !path) fail(LSG_EINVAL, "write_snapshot: null path");
            join_comm(s);
            std::vector<double> host(s->ctx->rank == 0 ? n : 0);
            gather_to_root(s->ctx, &s->g, s->slabs[0].f[s->cur], nullptr, host.data());
            if (s->ctx->rank == 0) {
                const int rc = lsg_write_snapshot(&s->g, host.data(), time, path);
                if (rc) fail(rc, g_err);
            }
            return;
        }
        if (!path) fail(LSG_EINVAL, "write_snapshot: null path");
        std::vector<double> host(n);
        download(s, host.data(), s->cur);
        const int rc = lsg_write_snapshot(&s->g, host.data(), time, path);
        if (rc) fail(rc, g_err);
    });
}

int lsg_gather_field(lsg_ctx* ctx, const lsg_grid* g, const double* local, double* global_out) {
    return guarded([&] {
        activate(ctx);
        check_grid(g);
        if (!local) fail(LSG_EINVAL, "gather_field: null local slab");
        if (ctx->nranks <= 1 || !ctx->comm) {  // one rank: the slab is the field
            if (!global_out) fail(LSG_EINVAL, "gather_field: null output");
            if (global_out != local) std::memcpy(global_out, local, sizeof(double) * static_cast<size_t>(node_count(g)));
            return;
        }
        if (ctx->rank == 0 && !global_out) fail(LSG_EINVAL, "gather_field: null output on rank 0");
        gather_to_root(ctx, g, nullptr, local, global_out);
    });
}

int lsg_solver_stream(lsg_solver* s, void** stream) {
    return guarded([&] {
        if (!s || !stream) fail(LSG_EINVAL, "stream: null argument");
        *stream = reinterpret_cast<void*>(s->ctx->stream);
    });
}

int lsg_probe_fp64_rate(lsg_ctx* ctx, double* instr_per_s) {
    return guarded([&] {
        if (!instr_per_s) fail(LSG_EINVAL, "probe: null output");
        activate(ctx);
        int sms = 0;
        CUDA_CHECK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, ctx->device));
        const int blocks = sms * 8, iters = 4000;
        DevBuf out;
        out.alloc(sizeof(double) * static_cast<size_t>(blocks) * 256, ctx->stream);
        cudaEvent_t e0, e1;
        CUDA_CHECK(cudaEventCreate(&e0));
        CUDA_CHECK(cudaEventCreate(&e1));
        double best = 0.0;
        for (int rep = 0; rep < 3; ++rep) {  // the first run warms clocks and caches
            CUDA_CHECK(cudaEventRecord(e0, ctx->stream));
            launch_fp64_rate(out.as<double>(), blocks, iters, ctx->stream);
            ctx->note_launch();
            CUDA_CHECK(cudaEventRecord(e1, ctx->stream));
            CUDA_CHECK(cudaEventSynchronize(e1));
            float ms = 0.f;
            CUDA_CHECK(cudaEventElapsedTime(&ms, e0, e1));
            const double ops = static_cast<double>(blocks) * 256.0 * iters * 8.0;
            if (rep > 0) best = std::max(best, ops / (ms * 1e-3));
        }
        cudaEventDestroy(e0);
        cudaEventDestroy(e1);
        out.release();
        *instr_per_s = best;
    });
}

int lsg_ctx_comm_info(const lsg_ctx* ctx, int* nranks, int* rank) {
    return guarded([&] {
        if (!ctx || !nranks || !rank) fail(LSG_EINVAL, "comm_info: null argument");
        *nranks = 0;
        *rank = -1;
        if (ctx->comm) {
            NCCL_CHECK(ncclCommCount(ctx->comm, nranks));
            NCCL_CHECK(ncclCommUserRank(ctx->comm, rank));
        }
    });
}

int lsg_solver_launches_per_step(const lsg_solver* s, int* n) {
    return guarded([&] {
        if (!s || !n) fail(LSG_EINVAL, "launches_per_step: null argument");
        int per_stage = 0;  // one launch, or boundary bands + interior (run_stage)
        for (const Slab& sl : s->slabs)
            per_stage += (s->halo_w == 0 || !s->overlap_halo) ? 1 : (sl.nz > 2 * s->halo_w ? 2 : 1);
        *n = stages_of(s->method) * per_stage;
    });
}

}  // extern "C"
