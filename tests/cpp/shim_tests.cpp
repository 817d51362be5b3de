// tests/cpp/shim_tests.cpp — the reference's own doctest cases
// (/root/reference/proj/tests/test_*.cpp), re-expressed against the C++ drop-in
// layer (include/levelset_b200/levelset.hpp), i.e. reference-style call sites
// compiled unchanged except for the header and the device Hamiltonian.
// Run by tests/test_gpu_shim.py on the GPU box; prints one line per failure.
#include <array>
#include <cmath>
#include <cstdio>
#include <limits>
#include <numbers>
#include <random>
#include <stdexcept>
#include <vector>

#include "levelset_b200/levelset.hpp"

using namespace levelset;

static int g_checks = 0, g_fail = 0;
#define CHECK(cond)                                                          \
    do {                                                                     \
        ++g_checks;                                                          \
        if (!(cond)) {                                                       \
            ++g_fail;                                                        \
            std::printf("FAIL %s:%d: %s\n", __FILE__, __LINE__, #cond);      \
        }                                                                    \
    } while (0)
#define CHECK_THROWS_AS(expr, E)                                             \
    do {                                                                     \
        ++g_checks;                                                          \
        bool ok_ = false;                                                    \
        try {                                                                \
            (void)(expr);                                                    \
        } catch (const E&) {                                                 \
            ok_ = true;                                                      \
        } catch (...) {                                                      \
        }                                                                    \
        if (!ok_) {                                                          \
            ++g_fail;                                                        \
            std::printf("FAIL %s:%d: %s does not throw %s\n", __FILE__, __LINE__, #expr, #E); \
        }                                                                    \
    } while (0)
static bool approx(double a, double b, double eps) { return std::abs(a - b) <= eps * std::max(1.0, std::abs(b)); }

constexpr double two_pi = 2.0 * std::numbers::pi;
constexpr double inf = std::numeric_limits<double>::infinity();

static ScalarField random_field(GridPtr g, std::uint64_t seed) {
    std::mt19937_64 rng(seed);
    std::uniform_real_distribution<double> dist(-1.0, 1.0);
    ScalarField f(g);
    for (std::size_t i = 0; i < f.size(); ++i) f[i] = dist(rng);
    return f;
}

static HamiltonianProblem advection_problem(GridPtr g, std::vector<double> u,
                                            DerivativeScheme s = DerivativeScheme::Eno2) {
    HamiltonianProblem p;
    p.grid = g;
    p.costate_scheme = s;
    p.device = linear_hamiltonian(u);
    return p;
}

static void grid_tests() {  // test_grid.cpp:96-202
    auto g = Grid::create({0.0}, {3.0}, {4}, {0});
    ScalarField f(g, std::vector<double>{1.0, 2.0, 3.0, 4.0});
    const PaddedField p = pad_ghost(f, 0, 1);
    const std::vector<double> e{4.0, 1.0, 2.0, 3.0, 4.0, 1.0};
    CHECK(p.data == e);
    auto g2 = Grid::create({0.0}, {3.0}, {4});
    ScalarField f2(g2, std::vector<double>{0.0, 1.0, 2.0, 3.0});
    const std::vector<double> e2{-2.0, -1.0, 0.0, 1.0, 2.0, 3.0, 4.0, 5.0};
    CHECK(pad_ghost(f2, 0, 2).data == e2);
    const ScalarField plus = shift_along_dim(p, 1);
    CHECK(plus[0] == 2.0 && plus[3] == 1.0);
    CHECK_THROWS_AS(shift_along_dim(p, 2), std::invalid_argument);
    auto g3 = Grid::create({0.0}, {1.0}, {4});
    ScalarField f3(g3);
    CHECK_THROWS_AS(pad_ghost(f3, 0, 4), std::invalid_argument);
    CHECK_THROWS_AS(pad_ghost(f3, 0, 0), std::invalid_argument);
    CHECK_THROWS_AS(pad_ghost(f3, 1, 1), std::invalid_argument);
    CHECK_THROWS_AS(Grid::create({0.0}, {1.0}, {2}), std::invalid_argument);
    CHECK_THROWS_AS(ScalarField(g3, std::vector<double>{1.0}), std::invalid_argument);
    auto g4 = Grid::create({0.0, 0.0}, {1.0, 2.0}, {8, 5}, {0, 1});
    const ScalarField r = random_field(g4, 99);
    for (int dim = 0; dim < 2; ++dim)
        for (int off : {-2, -1, 1, 2}) {
            const ScalarField s = shift_along_dim(pad_ghost(r, dim, 2), off);
            const ScalarField b = shift_along_dim(pad_ghost(s, dim, 2), -off);
            bool same = true;
            for (std::size_t i = 0; i < r.size(); ++i) same = same && b[i] == r[i];
            CHECK(same);
        }
}

static void derivative_tests() {  // test_spatial_derivatives.cpp:58-237
    auto g = Grid::create({0.0}, {2.0}, {5});
    ScalarField v(g);
    for (std::size_t i = 0; i < v.size(); ++i) v[i] = g->axis(0)[i] * g->axis(0)[i];
    const DerivativePair d = upwind_first_first(v, 0);
    CHECK(d.dim == 0 && approx(d.left[2], 1.5, 1e-14) && approx(d.right[2], 2.5, 1e-14));
    auto gl = Grid::create({-1.0}, {1.0}, {9});
    ScalarField lin(gl);
    for (std::size_t i = 0; i < lin.size(); ++i) lin[i] = 3.0 * gl->axis(0)[i];
    for (DerivativeScheme s : {DerivativeScheme::First, DerivativeScheme::Eno2, DerivativeScheme::Eno3,
                               DerivativeScheme::Weno5}) {
        const DerivativePair dl = upwind_derivative(lin, 0, s);
        bool ok = true;
        for (std::size_t i = 0; i < lin.size(); ++i) ok = ok && approx(dl.left[i], 3.0, 1e-12) && approx(dl.right[i], 3.0, 1e-12);
        CHECK(ok);
    }
    auto gs = Grid::create({0.0}, {7.0}, {8});
    const ScalarField step(gs, std::vector<double>{0, 0, 0, 0, 1, 1, 1, 1});
    const DerivativePair e2 = upwind_first_eno2(step, 0);
    CHECK(std::abs(e2.left[6]) <= 1e-14 && std::abs(e2.right[5]) <= 1e-14);
    auto gc = Grid::create({-1.0}, {1.0}, {33});
    ScalarField cub(gc);
    for (std::size_t i = 0; i < cub.size(); ++i) cub[i] = std::pow(gc->axis(0)[i], 3);
    const DerivativePair e3 = upwind_first_eno3(cub, 0);
    bool ok3 = true;
    for (std::size_t i = 3; i + 3 < cub.size(); ++i) {
        const double x = gc->axis(0)[i];
        ok3 = ok3 && approx(e3.left[i], 3 * x * x, 1e-10) && approx(e3.right[i], 3 * x * x, 1e-10);
    }
    CHECK(ok3);
    for (bool periodic : {false, true}) {  // bitwise axis reversal :194-213
        auto gr = periodic ? Grid::create({-1.0}, {1.0}, {24}, {0}) : Grid::create({-1.0}, {1.0}, {24});
        const ScalarField a = random_field(gr, 41);
        ScalarField w(gr);
        const std::size_t n = a.size();
        for (std::size_t i = 0; i < n; ++i) w[i] = a[n - 1 - i];
        for (DerivativeScheme s : {DerivativeScheme::First, DerivativeScheme::Eno2, DerivativeScheme::Eno3,
                                   DerivativeScheme::Weno5}) {
            const DerivativePair dv = upwind_derivative(a, 0, s), dw = upwind_derivative(w, 0, s);
            bool same = true;
            for (std::size_t i = 0; i < n; ++i) same = same && dw.left[i] == -dv.right[n - 1 - i] && dw.right[i] == -dv.left[n - 1 - i];
            CHECK(same);
        }
    }
    auto tiny = Grid::create({0.0}, {1.0}, {5});
    const ScalarField z(tiny, 0.0);
    CHECK_THROWS_AS(upwind_first_eno3(z, 0), std::invalid_argument);
    CHECK_THROWS_AS(upwind_first_weno5(z, 0), std::invalid_argument);
    CHECK_THROWS_AS(upwind_first_first(z, 1), std::invalid_argument);
}

static void hamiltonian_tests() {  // test_hamiltonian.cpp:40-193
    auto g = Grid::create({0.0}, {1.0 - 1.0 / 128.0}, {128}, {0});
    ScalarField v(g);
    for (std::size_t i = 0; i < v.size(); ++i) v[i] = std::sin(two_pi * g->axis(0)[i]);
    const TermResult adv = term_lax_friedrichs(0.0, v, advection_problem(g, {0.7}));
    bool ok = true;
    for (std::size_t i = 0; i < v.size(); ++i) ok = ok && approx(adv.dvdt[i], -0.7 * two_pi * std::cos(two_pi * g->axis(0)[i]), 5e-3 * 5);
    CHECK(ok);
    auto g11 = Grid::create({0.0}, {1.0}, {11});
    CHECK(approx(term_lax_friedrichs(0.0, ScalarField(g11, 0.0), advection_problem(g11, {2.0})).step_bound, 0.05, 1e-14));
    CHECK(term_lax_friedrichs(0.0, ScalarField(g11, 0.0), advection_problem(g11, {0.0})).step_bound == inf);
    auto g5 = Grid::create({0.0}, {2.0}, {5});
    ScalarField sq(g5);
    for (std::size_t i = 0; i < sq.size(); ++i) sq[i] = g5->axis(0)[i] * g5->axis(0)[i];
    HamiltonianProblem pc = advection_problem(g5, {1.0}, DerivativeScheme::First);
    pc.device = linear_hamiltonian({1.0}, {0.0});
    CHECK(approx(term_lax_friedrichs(0.0, sq, pc).dvdt[2], -2.0, 1e-14));
    auto g17 = Grid::create({0.0}, {1.0}, {17});
    ScalarField dy(g17);
    for (std::size_t i = 0; i < dy.size(); ++i) dy[i] = 1.5 * g17->axis(0)[i];
    HamiltonianProblem pd;
    pd.grid = g17;
    pd.device = linear_hamiltonian({0.25}, {0.25}, 0.125);
    const TermResult rd = term_lax_friedrichs(0.0, dy, pd);
    bool exact = true;
    for (std::size_t i = 0; i < dy.size(); ++i) exact = exact && rd.dvdt[i] == -(0.25 * 1.5 + 0.125);
    CHECK(exact);
    auto g3 = Grid::create({0.0}, {1.0}, {3});
    const ScalarField dv3(g3, std::vector<double>{-2.0, 0.0, 3.0});
    const ScalarField grow = restrict_update(dv3, UpdateDirection::Grow);
    const ScalarField shrink = restrict_update(dv3, UpdateDirection::Shrink);
    CHECK(grow[0] == -2.0 && grow[1] == 0.0 && grow[2] == 0.0);
    CHECK(shrink[0] == 0.0 && shrink[1] == 0.0 && shrink[2] == 3.0);
    auto g32 = Grid::create({0.0}, {1.0 - 1.0 / 32.0}, {32}, {0});
    ScalarField s32(g32);
    for (std::size_t i = 0; i < s32.size(); ++i) s32[i] = std::sin(two_pi * g32->axis(0)[i]);
    HamiltonianProblem pcl = advection_problem(g32, {1.0});
    pcl.restrict_update = true;
    const TermResult clamped = term_lax_friedrichs(0.0, s32, pcl);
    pcl.restrict_update = false;
    const TermResult free_run = term_lax_friedrichs(0.0, s32, pcl);
    bool clamp_ok = true, any_pos = false;
    for (std::size_t i = 0; i < s32.size(); ++i) {
        clamp_ok = clamp_ok && clamped.dvdt[i] == std::min(free_run.dvdt[i], 0.0);
        any_pos = any_pos || free_run.dvdt[i] > 0.0;
    }
    CHECK(clamp_ok && any_pos && clamped.step_bound == free_run.step_bound);
    HamiltonianProblem nanp = advection_problem(g5, {std::numeric_limits<double>::quiet_NaN()}, DerivativeScheme::Eno2);
    nanp.device = linear_hamiltonian({std::numeric_limits<double>::quiet_NaN()}, {1.0});
    CHECK_THROWS_AS(term_lax_friedrichs(0.0, ScalarField(g5, 1.0), nanp), std::runtime_error);
    HamiltonianProblem badb = advection_problem(g5, {1.0});
    badb.device = linear_hamiltonian({1.0}, {-1.0});
    CHECK_THROWS_AS(term_lax_friedrichs(0.0, ScalarField(g5, 1.0), badb), std::runtime_error);
    HamiltonianProblem host_only;
    host_only.grid = g5;
    host_only.ham_func = [](double, const Grid&, std::span<const ScalarField>, ScalarField&) {};
    CHECK_THROWS_AS(term_lax_friedrichs(0.0, ScalarField(g5, 1.0), host_only), std::invalid_argument);
    CHECK_THROWS_AS(term_lax_friedrichs(0.0, ScalarField(g11, 1.0), advection_problem(g5, {1.0})), std::invalid_argument);
}

static void integrator_tests() {  // test_integrator.cpp:111-244
    auto g = Grid::create({0.0}, {1.0 - 1.0 / 64.0}, {64}, {0});
    ScalarField v0(g);
    for (std::size_t i = 0; i < v0.size(); ++i) v0[i] = std::sin(two_pi * g->axis(0)[i]);
    const TermFn term = make_lax_friedrichs_term(advection_problem(g, {1.0}, DerivativeScheme::First));
    IntegratorOptions opts;
    opts.cfl_factor = 0.5;
    opts.max_step = 0.009;
    const IntegrationResult r = ode_cfl_3(term, {0.0, 0.25}, v0, opts);
    CHECK(r.t == 0.25 && !r.steps.empty());
    double t_expect = 0.0;
    bool ok = true;
    for (const StepLogEntry& e : r.steps) {
        ok = ok && e.t == t_expect && e.dt > 0.0 && e.dt <= opts.cfl_factor * e.step_bound && e.dt <= opts.max_step;
        t_expect = e.t + e.dt;
    }
    CHECK(ok);
    IntegratorOptions ck;
    ck.max_step = 0.01;
    ck.checkpoint_times = {0.03, 0.077};
    const IntegrationResult rc = ode_cfl_1(term, {0.0, 0.1}, v0, ck);
    bool hit1 = false, hit2 = false;
    for (const StepLogEntry& e : rc.steps) {
        hit1 = hit1 || e.t == 0.03;
        hit2 = hit2 || e.t == 0.077;
    }
    CHECK(rc.t == 0.1 && hit1 && hit2);
    const IntegrationResult a = ode_cfl_3(term, {0.0, 0.5}, v0), b = ode_cfl_3(term, {0.0, 0.5}, v0);
    bool det = a.steps.size() == b.steps.size() && a.t == b.t;
    for (std::size_t i = 0; det && i < a.v.size(); ++i) det = a.v[i] == b.v[i];
    CHECK(det);
    const IntegrationResult z = ode_cfl_2(term, {4.0, 4.0}, v0);
    CHECK(z.t == 4.0 && z.steps.empty() && z.v[3] == v0[3]);
    IntegratorOptions bad;
    bad.cfl_factor = 0.0;
    CHECK_THROWS_AS(ode_cfl_1(term, {0.0, 1.0}, v0, bad), std::invalid_argument);
    bad = {};
    bad.checkpoint_times = {0.5, 0.2};
    CHECK_THROWS_AS(ode_cfl_1(term, {0.0, 1.0}, v0, bad), std::invalid_argument);
    CHECK_THROWS_AS(ode_cfl_1(term, {1.0, 0.0}, v0), std::invalid_argument);
    CHECK_THROWS_AS(ode_cfl_1(term, {0.0, inf}, v0), std::invalid_argument);
    const TermFn host_lambda = [](double, const ScalarField& v) { return TermResult{ScalarField(v.grid_ptr(), 0.0), 1.0}; };
    CHECK_THROWS_AS(ode_cfl_1(host_lambda, {0.0, 1.0}, v0), std::invalid_argument);
}

static void reachability_tests() {  // test_reachability.cpp:59-285, acceptance.cpp:381-419
    const RocketParams prm;
    CHECK(rocket_hamiltonian_value(13.0, 0.7, 0.0, 0.0, 0.0, prm) == 0.0);
    CHECK(approx(rocket_hamiltonian_value(0.0, 0.0, 0.0, 0.0, 1.0, prm), -2.0, 1e-15));
    const ProblemSetup setup = build_rocket_problem(9);
    const Grid& g = *setup.problem.grid;
    CHECK(g.dim() == 3 && g.min(0) == -64.0 && g.count(2) == 9);
    CHECK(setup.problem.costate_scheme == DerivativeScheme::Eno2 && setup.problem.restrict_update);
    CHECK(approx(setup.initial_value[g.index(std::vector<int>{4, 4, 0})], -1.5, 1e-15));
    CHECK(approx(setup.initial_value[g.index(std::vector<int>{6, 4, 3})], 32.0 - 1.5, 1e-15));
    CHECK_THROWS_AS(build_rocket_problem(5), std::invalid_argument);
    const SolveOutcome out = solve_brt(setup, {-0.1, 0.0}, 3);
    CHECK(out.checkpoints.size() == 3 && out.checkpoint_times[0] == 0.0 && approx(out.checkpoint_times[2], 0.1, 1e-15));
    CHECK(!out.steps.empty() && out.integration_seconds > 0.0);
    bool mono = true;
    for (std::size_t k = 1; k < out.checkpoints.size(); ++k)
        for (std::size_t i = 0; i < setup.initial_value.size(); ++i) mono = mono && out.checkpoints[k][i] <= out.checkpoints[k - 1][i];
    CHECK(mono);
    const SolveOutcome zero = solve_brt(setup, {0.0, 0.0}, 5);
    CHECK(zero.checkpoints.size() == 1 && zero.steps.empty());
    CHECK_THROWS_AS(solve_brt(setup, {0.0, 1.0}, 0), std::invalid_argument);
    ProblemSetup mismatched = build_rocket_problem(9);
    mismatched.initial_value = ScalarField(build_rocket_problem(11).problem.grid);
    CHECK_THROWS_AS(solve_brt(mismatched, {0.0, 1.0}, 2), std::invalid_argument);
    // acceptance criterion 5: rockets N = 50 over (-2.5, 0) with 11 checkpoints takes 490 steps
    const SolveOutcome big = solve_brt(build_rocket_problem(50), {-2.5, 0.0}, 11);
    CHECK(big.steps.size() == 490 && big.checkpoints.size() == 11);
    const ProblemSetup rot = rigid_rotation_problem(21);
    CHECK(approx(rot.initial_value[rot.problem.grid->index(std::vector<int>{15, 10})], -0.5, 1e-15));
    const SolveOutcome ro = solve_brt(rot, {0.0, 0.5}, 2);
    double vmin = ro.checkpoints[1][0], vmax = vmin;
    for (double x : ro.checkpoints[1].values()) vmin = std::min(vmin, x), vmax = std::max(vmax, x);
    CHECK(vmin < -0.3 && vmin > -0.7 && vmax > 0.5);
    bool cfl = true;
    for (const StepLogEntry& e : ro.steps) cfl = cfl && e.dt <= 0.32 * e.step_bound;
    CHECK(cfl);
}

static void contour_tests() {  // contour.cpp via the drop-in
    const ProblemSetup rot = rigid_rotation_problem(101);
    const auto segs = extract_zero_set_2d(rot.initial_value);
    CHECK(!segs.empty());
    const double len = polyline_length(segs);
    CHECK(std::abs(len - 2.0 * std::numbers::pi * 0.5) < 0.01);  // circle of radius 0.5
    const ProblemSetup rk = build_rocket_problem(21);
    const ScalarField sl = slice_2d(rk.initial_value, 2, 3);
    CHECK(sl.grid().dim() == 2 && sl.size() == 21u * 21u);
    CHECK_THROWS_AS(extract_zero_set_2d(rk.initial_value), std::invalid_argument);
}

// test_implicit_surfaces.cpp:66-150 re-expressed against the drop-in
static void implicit_surface_tests() {
    auto node = [](const Grid& g, std::initializer_list<int> m) { return g.index(std::vector<int>(m)); };
    {
        auto g = Grid::create({-2.0, -2.0}, {2.0, 2.0}, {5, 5});
        const ScalarField v = rectangle(g, {-1.0, -1.0}, {1.0, 1.0});
        CHECK(approx(v[node(*g, {2, 2})], -1.0, 1e-14));
        CHECK(approx(v[node(*g, {4, 2})], 1.0, 1e-14));
        CHECK(approx(v[node(*g, {3, 3})], 0.0, 1e-14));
        CHECK(approx(v[node(*g, {4, 4})], 1.0, 1e-14));
        CHECK_THROWS_AS(rectangle(g, {1.0, -1.0}, {-1.0, 1.0}), std::invalid_argument);
    }
    {
        auto g2 = Grid::create({-3.0, -3.0}, {3.0, 3.0}, {7, 7});
        const ScalarField e2 = ellipsoid(g2, 4.0);
        CHECK(approx(e2[node(*g2, {3, 3})], -4.0, 1e-14));
        CHECK(approx(e2[node(*g2, {3, 4})], 0.0, 1e-14));
        CHECK(approx(e2[node(*g2, {5, 3})], 0.0, 1e-14));
        auto g3 = Grid::create({-3.0, -3.0, -3.0}, {3.0, 3.0, 3.0}, {7, 7, 7});
        const ScalarField e3 = ellipsoid(g3, 9.0);
        CHECK(approx(e3[node(*g3, {3, 3, 4})], 0.0, 1e-14));
        CHECK(approx(e3[node(*g3, {6, 3, 3})], 0.0, 1e-14));
        auto g1 = Grid::create({0.0}, {1.0}, {5});
        CHECK_THROWS_AS(ellipsoid(g1, 1.0), std::invalid_argument);
    }
    {
        auto g = Grid::create({-2.0, -2.0, -2.0}, {2.0, 2.0, 2.0}, {5, 5, 5});
        const ScalarField a = sphere(g, {-1.0, 0.0, 0.0}, 1.0);
        const ScalarField b = sphere(g, {1.0, 0.0, 0.0}, 1.0);
        const ScalarField u = set_union(a, b);
        const ScalarField n = set_intersection(a, b);
        bool ok = true;
        for (std::size_t i = 0; i < u.size(); ++i)
            ok = ok && u[i] == std::min(a[i], b[i]) && n[i] == std::max(a[i], b[i]);
        CHECK(ok);
        CHECK(approx(u[node(*g, {1, 2, 2})], -1.0, 1e-14));
        CHECK(approx(u[node(*g, {2, 2, 2})], 0.0, 1e-14));
        const ScalarField c = set_complement(a);
        const ScalarField cc = set_complement(c);
        ok = true;
        for (std::size_t i = 0; i < c.size(); ++i) ok = ok && c[i] == -a[i] && cc[i] == a[i];
        CHECK(ok);
    }
    {  // De Morgan bit for bit
        auto g = Grid::create({-2.0, -2.0, -2.0}, {2.0, 2.0, 2.0}, {9, 9, 9});
        std::mt19937_64 rng(2024);
        std::uniform_real_distribution<double> center(-1.5, 1.5), radius(0.2, 2.0);
        bool ok = true;
        for (int trial = 0; trial < 10; ++trial) {
            const ScalarField a = sphere(g, {center(rng), center(rng), center(rng)}, radius(rng));
            const double lo = center(rng);
            const ScalarField b = rectangle(g, {lo, lo, lo}, {lo + radius(rng), lo + radius(rng), lo + radius(rng)});
            const ScalarField lhs = set_complement(set_union(a, b));
            const ScalarField rhs = set_intersection(set_complement(a), set_complement(b));
            const ScalarField lhs2 = set_complement(set_intersection(a, b));
            const ScalarField rhs2 = set_union(set_complement(a), set_complement(b));
            for (std::size_t i = 0; i < lhs.size(); ++i) ok = ok && lhs[i] == rhs[i] && lhs2[i] == rhs2[i];
        }
        CHECK(ok);
    }
    {
        auto g1 = Grid::create({-2.0, -2.0, -2.0}, {2.0, 2.0, 2.0}, {5, 5, 5});
        auto g2 = Grid::create({-2.0, -2.0, -2.0}, {2.0, 2.0, 2.0}, {5, 5, 5});
        const ScalarField a = sphere(g1, {0.0, 0.0, 0.0}, 1.0);
        const ScalarField b = sphere(g2, {0.0, 0.0, 0.0}, 1.0);
        CHECK_THROWS_AS(set_union(a, b), std::invalid_argument);
        CHECK_THROWS_AS(set_intersection(a, b), std::invalid_argument);
    }
}

// reachability.hpp plugins on the device (test_reachability.cpp:115-143 re-expressed
// for the closed form) and detail::fill_padded_line
static void plugin_tests() {
    const RocketParams prm;
    auto g = Grid::create({-64.0, -64.0, -4.0}, {64.0, 64.0, 4.0}, {9, 9, 9});
    std::array<ScalarField, 3> bounds = {ScalarField(g), ScalarField(g), ScalarField(g)};
    for (int d = 0; d < 3; ++d) rocket_dissipation(0.0, *g, d, bounds[static_cast<std::size_t>(d)], prm);
    std::mt19937_64 rng(47);
    std::uniform_real_distribution<double> costate(-3.0, 3.0);
    std::vector<ScalarField> cs = {ScalarField(g), ScalarField(g), ScalarField(g)};
    for (auto& c : cs)
        for (std::size_t i = 0; i < c.size(); ++i) c[i] = costate(rng);
    ScalarField h(g);
    rocket_hamiltonian(0.0, *g, std::span<const ScalarField>(cs), h, prm);
    const double eps = 1e-6;
    bool dominated = true, exact = true;
    for (std::size_t i = 0; i < g->node_count(); ++i) {
        const double x = g->coords(0)[i], th = g->coords(2)[i];
        const double p1 = cs[0][i], p2 = cs[1][i], p3 = cs[2][i];
        exact = exact && h[i] == rocket_hamiltonian_value(x, th, p1, p2, p3, prm);  // same bits
        for (int d = 0; d < 3; ++d) {
            const double q1 = p1 + (d == 0 ? eps : 0.0), q2 = p2 + (d == 1 ? eps : 0.0), q3 = p3 + (d == 2 ? eps : 0.0);
            const double slope = std::abs(rocket_hamiltonian_value(x, th, q1, q2, q3, prm) -
                                          rocket_hamiltonian_value(x, th, p1, p2, p3, prm)) / eps;
            dominated = dominated && slope <= bounds[static_cast<std::size_t>(d)][i] + 1e-6;
        }
    }
    CHECK(exact);
    CHECK(dominated);
    CHECK_THROWS_AS(rocket_dissipation(0.0, *g, 3, bounds[0], prm), std::invalid_argument);
    // the plugins a device problem carries evaluate the same thing
    const ProblemSetup setup = build_rocket_problem(9);
    const Grid& rg = *setup.problem.grid;
    std::vector<ScalarField> rcs = {random_field(setup.problem.grid, 1), random_field(setup.problem.grid, 2),
                                    random_field(setup.problem.grid, 3)};
    ScalarField a(setup.problem.grid), b(setup.problem.grid);
    setup.problem.ham_func(0.0, rg, std::span<const ScalarField>(rcs), a);
    rocket_hamiltonian(0.0, rg, std::span<const ScalarField>(rcs), b, prm);
    bool same = true;
    for (std::size_t i = 0; i < a.size(); ++i) same = same && a[i] == b[i];
    CHECK(same);
    setup.problem.dissipation_bounds(0.0, rg, 1, a);
    rocket_dissipation(0.0, rg, 1, b, prm);
    same = true;
    for (std::size_t i = 0; i < a.size(); ++i) same = same && a[i] == b[i];
    CHECK(same);
    // detail::fill_padded_line == the matching line of pad_ghost
    auto g2 = Grid::create({-1.0, -1.0}, {1.0, 1.0}, {11, 7}, {1});
    const ScalarField f = random_field(g2, 9);
    for (int dim = 0; dim < 2; ++dim) {
        const PaddedField pf = pad_ghost(f, dim, 3);
        const int n = g2->count(dim);
        const std::size_t stride = dim == 0 ? 1 : 11;
        std::vector<double> dst(static_cast<std::size_t>(n + 6));
        detail::fill_padded_line(f.values(), 2 * (dim == 0 ? 11 : 1), stride, n, 3, g2->boundary(dim), dst);
        bool ok = true;
        for (int j = 0; j < n + 6; ++j) {
            const std::size_t base = dim == 0 ? 2 * (n + 6) : 2;
            ok = ok && dst[static_cast<std::size_t>(j)] == pf.data[base + static_cast<std::size_t>(j) * stride];
        }
        CHECK(ok);
    }
}

static void convergence_table_tests() {  // expected text: the reference's format_convergence_table
    const std::vector<ConvergenceRow> rows = {{11, 0.2, 0.012345678901234, std::nan(""), false},
                                              {21, 0.1, 0.0031234, 1.98321, false},
                                              {41, 0.05, 1e-17, 2.0, true},
                                              {81, 0.025, 2e-17, 0.5, true}};
    CHECK(format_convergence_table(rows) ==
          "n,dx,max_error,order\n11,0.2,0.0123456789012,\n21,0.1,0.0031234,1.98321\n41,0.05,1e-17,2\n"
          "81,0.025,2e-17,exact\n");
}

int main() {
    try {
        convergence_table_tests();
        plugin_tests();
        implicit_surface_tests();
        grid_tests();
        derivative_tests();
        hamiltonian_tests();
        integrator_tests();
        reachability_tests();
        contour_tests();
    } catch (const std::exception& e) {
        std::printf("FAIL uncaught exception: %s\n", e.what());
        return 2;
    }
    std::printf("%d checks, %d failures\n", g_checks, g_fail);
    return g_fail ? 1 : 0;
}
