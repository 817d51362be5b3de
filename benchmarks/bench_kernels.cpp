// Kernel-level microbenchmarks: the reference's bench_kernels.cpp suite
// (proj/benchmarks/bench_kernels.cpp:33-117: pad_ghost, the four one-sided
// derivative schemes, the rockets Lax-Friedrichs term, one RK3 step of the
// rockets and rigid-rotation problems, same sizes and seeds) as ONE source
// compiled twice:
//
//   -DLSG_B200  against the C++ drop-in (include/levelset_b200/levelset.hpp,
//               liblevelset_b200.so) -> benchmarks/bench_kernels_b200
//   otherwise   against the reference's own headers and sources
//               (oracle/Makefile)                 -> oracle/_ref/bench_kernels_ref
//
// google-benchmark is not in the image, so the timing loop is a small
// stand-in with the same semantics (warm-up, iterate to a minimum time,
// items/s = nodes per iteration).  Every case also prints a checksum of its
// output (hex-float sum in index order) so the two builds can be compared
// bit for bit.  Host buffers in and out on every call: this is the
// reference-facing API, host<->device copies included.
#include <chrono>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <functional>
#include <numbers>
#include <random>
#include <span>
#include <string>
#include <vector>

#ifdef LSG_B200
#include "levelset_b200/levelset.hpp"
#define IMPL "b200"
#else
#include "levelset/grid.hpp"
#include "levelset/hamiltonian.hpp"
#include "levelset/integrator.hpp"
#include "levelset/reachability.hpp"
#include "levelset/spatial_derivatives.hpp"
#define IMPL "reference"
#endif

using namespace levelset;

namespace {

double g_min_time = 0.5;

ScalarField random_field(GridPtr grid, std::uint64_t seed) {
    std::mt19937_64 rng(seed);
    std::uniform_real_distribution<double> dist(-1.0, 1.0);
    ScalarField f(grid);
    for (std::size_t i = 0; i < f.size(); ++i) f[i] = dist(rng);
    return f;
}

GridPtr cube_grid(int n) { return Grid::create({-1.0, -1.0, -1.0}, {1.0, 1.0, 1.0}, {n, n, n}, {2}); }

double checksum(std::span<const double> x) {
    double s = 0.0;
    for (double v : x) s += v;
    return s;
}

TermFn lf_term(const HamiltonianProblem& problem) {
#ifdef LSG_B200
    return make_lax_friedrichs_term(problem);  // the one call-site edit
#else
    return [&problem](double t, const ScalarField& f) { return term_lax_friedrichs(t, f, problem); };
#endif
}

// Run `body` until g_min_time has elapsed; body(true) also returns the output
// checksum (warm-up call only, so the sum stays out of the timed loop).
void run(const std::string& name, long long items, const std::function<double(bool)>& body) {
    const double sum = body(true);
    long long iters = 0;
    const auto t0 = std::chrono::steady_clock::now();
    double el = 0.0;
    while (el < g_min_time || iters < 3) {
        body(false);
        ++iters;
        el = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    }
    const double ns = el / static_cast<double>(iters) * 1e9;
    std::printf("{\"impl\": \"%s\", \"name\": \"%s\", \"ns_per_iter\": %.1f, \"items_per_s\": %.6g, "
                "\"iters\": %lld, \"checksum\": \"%a\"}\n",
                IMPL, name.c_str(), ns, items > 0 ? static_cast<double>(items) / (ns * 1e-9) : 0.0, iters, sum);
    std::fflush(stdout);
}

void bench_pad_ghost(int n) {
    const ScalarField v = random_field(cube_grid(n), 1);
    run("bench_pad_ghost/" + std::to_string(n), static_cast<long long>(v.size()), [&](bool sum) {
        PaddedField padded = pad_ghost(v, 1, 3);
        return sum ? checksum(padded.data) : 0.0;
    });
}

void bench_derivative(const char* label, DerivativeScheme scheme, int n) {
    const ScalarField v = random_field(cube_grid(n), 2);
    run(std::string(label) + "/" + std::to_string(n), static_cast<long long>(v.size()), [&](bool sum) {
        DerivativePair d = upwind_derivative(v, 0, scheme);
        return sum ? checksum(d.left.values()) + checksum(d.right.values()) : 0.0;
    });
}

void bench_rocket_term(int n) {
    const ProblemSetup setup = build_rocket_problem(n);
    const ScalarField& v = setup.initial_value;
    run("bench_rocket_term/" + std::to_string(n), static_cast<long long>(v.size()), [&](bool sum) {
        TermResult r = term_lax_friedrichs(0.0, v, setup.problem);
        return sum ? checksum(r.dvdt.values()) + r.step_bound : 0.0;
    });
}

void bench_rk3_step(const char* label, const ProblemSetup& setup, int n) {
    const TermFn term = lf_term(setup.problem);
    IntegratorOptions opts;
    opts.max_step = 1e-3;  // one short step per iteration
    run(std::string(label) + "/" + std::to_string(n), static_cast<long long>(setup.initial_value.size()), [&](bool sum) {
        IntegrationResult r = ode_cfl_3(term, {0.0, opts.max_step}, setup.initial_value, opts);
        return sum ? checksum(r.v.values()) : 0.0;
    });
}

}  // namespace

int main(int argc, char** argv) {
    // --min-time S   (default 0.5 s per case)
    // --large        also run 128^3 / 101^3 / 201^2 sizes beyond the reference's own args
    bool large = false;
    for (int i = 1; i < argc; ++i) {
        if (!std::strcmp(argv[i], "--min-time") && i + 1 < argc) g_min_time = std::atof(argv[++i]);
        if (!std::strcmp(argv[i], "--large")) large = true;
    }
    std::vector<int> cube = {32, 64};
    if (large) cube.push_back(128);
    for (int n : cube) bench_pad_ghost(n);
    for (int n : cube) bench_derivative("bench_first", DerivativeScheme::First, n);
    for (int n : cube) bench_derivative("bench_eno2", DerivativeScheme::Eno2, n);
    for (int n : cube) bench_derivative("bench_eno3", DerivativeScheme::Eno3, n);
    for (int n : cube) bench_derivative("bench_weno5", DerivativeScheme::Weno5, n);
    std::vector<int> rk = {32, 50};
    if (large) rk.push_back(101);
    for (int n : rk) bench_rocket_term(n);
    for (int n : rk) bench_rk3_step("bench_rocket_rk3_step", build_rocket_problem(n), n);
    std::vector<int> rot = {101};
    if (large) rot.push_back(401);
    for (int n : rot) bench_rk3_step("bench_rotation_rk3_step", rigid_rotation_problem(n), n);
    return 0;
}
