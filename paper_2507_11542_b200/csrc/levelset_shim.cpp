// levelset_shim.cpp — the C++ drop-in layer (include/levelset_b200/levelset.hpp)
// over the C ABI (include/lsg.h).  Host bookkeeping only: every field
// operation is a device call; error codes are mapped back onto the exception
// types the reference throws.
#include "../../include/levelset_b200/levelset.hpp"

#include <cmath>
#include <cstring>
#include <iomanip>
#include <sstream>
#include <numbers>
#include <stdexcept>
#include <string>

#include "../../include/lsg.h"

namespace levelset {

namespace {

[[noreturn]] void rethrow(int rc) {
    const std::string msg = lsg_last_error();
    switch (rc) {
        case LSG_EINVAL: throw std::invalid_argument(msg);
        case LSG_ERANGE: throw std::out_of_range(msg);
        default: throw std::runtime_error(msg);
    }
}

void check(int rc) {
    if (rc != LSG_OK) rethrow(rc);
}

thread_local int t_device = 0;

struct CtxHolder {
    lsg_ctx* ctx = nullptr;
    int device = -1;
    ~CtxHolder() {
        if (ctx) lsg_ctx_destroy(ctx);
    }
};

lsg_ctx* ctx() {
    thread_local CtxHolder h;
    if (!h.ctx || h.device != t_device) {
        if (h.ctx) lsg_ctx_destroy(h.ctx);
        h.ctx = nullptr;
        check(lsg_ctx_create(t_device, &h.ctx));
        h.device = t_device;
    }
    return h.ctx;
}

lsg_grid to_c(const Grid& g) {
    if (g.dim() > LSG_MAX_DIM) throw std::invalid_argument("grid: the device path supports at most 6 dimensions");
    lsg_grid c{};
    c.dim = g.dim();
    for (int d = 0; d < g.dim(); ++d) {
        c.counts[d] = g.count(d);
        c.mins[d] = g.min(d);
        c.maxs[d] = g.max(d);
        if (g.boundary(d) == BoundaryCondition::Periodic) c.periodic_mask |= 1u << d;
    }
    return c;
}

int scheme_c(DerivativeScheme s) { return static_cast<int>(s); }

lsg_problem to_c(const HamiltonianProblem& p) {
    if (p.device.kind == 0)
        throw std::invalid_argument(
            "term_lax_friedrichs: problem has no device Hamiltonian (host std::function plugins cannot run on "
            "the B200 path)");
    lsg_problem c{};
    c.kind = p.device.kind;
    c.scheme = scheme_c(p.costate_scheme);
    c.direction = p.update_direction == UpdateDirection::Shrink ? LSG_SHRINK : LSG_GROW;
    c.restrict_update = p.restrict_update ? 1 : 0;
    c.options = static_cast<int>(p.options);
    for (int k = 0; k < LSG_MAX_PARAMS; ++k) c.params[k] = p.device.params[static_cast<std::size_t>(k)];
    return c;
}

struct OptsC {
    lsg_opts o{};
    explicit OptsC(const IntegratorOptions& opts) {
        o.cfl_factor = opts.cfl_factor;
        o.max_step = opts.max_step;
        o.termination_epsilon = opts.termination_epsilon;
        o.checkpoint_times = opts.checkpoint_times.empty() ? nullptr : opts.checkpoint_times.data();
        o.n_checkpoint_times = opts.checkpoint_times.size();
    }
};

std::vector<StepLogEntry> to_steps(const std::vector<lsg_steplog>& log, std::size_t n) {
    std::vector<StepLogEntry> out(n);
    for (std::size_t k = 0; k < n; ++k) out[k] = {log[k].t, log[k].dt, log[k].step_bound, log[k].v_min, log[k].v_max};
    return out;
}

// Device initial condition (lsg_solver_init_shape) on a scratch solver.
ScalarField device_shape(const GridPtr& grid, int shape, unsigned ignored, const std::vector<double>& center,
                         double radius, const std::vector<double>& upper = {}) {
    lsg_grid g = to_c(*grid);
    lsg_problem p{};
    p.kind = LSG_HAM_LINEAR;
    p.scheme = LSG_SCHEME_FIRST;
    lsg_solver* s = nullptr;
    check(lsg_solver_create(ctx(), &g, &p, LSG_CFL1, &s));
    double c[LSG_MAX_DIM] = {0, 0, 0, 0, 0, 0}, u[LSG_MAX_DIM] = {0, 0, 0, 0, 0, 0};
    for (std::size_t d = 0; d < center.size() && d < LSG_MAX_DIM; ++d) c[d] = center[d];
    for (std::size_t d = 0; d < upper.size() && d < LSG_MAX_DIM; ++d) u[d] = upper[d];
    ScalarField out(grid);
    int rc = lsg_solver_apply_shape(s, 0, shape, ignored, c, u, radius);
    if (rc == LSG_OK) rc = lsg_solver_get_field(s, out.values().data());
    lsg_solver_destroy(s);
    check(rc);
    return out;
}

// The device Hamiltonian / dissipation bound as host-callable plugins (the
// reference's HamiltonianFn / DissipationFn signatures), for problems built
// with a device kind.
void device_eval(const Grid& grid, const DeviceHamiltonian& dev, int dim, std::span<const ScalarField> costate,
                 ScalarField& out) {
    lsg_grid g = to_c(grid);
    lsg_problem p{};
    p.kind = dev.kind;
    p.scheme = LSG_SCHEME_FIRST;
    for (int k = 0; k < LSG_MAX_PARAMS; ++k) p.params[k] = dev.params[static_cast<std::size_t>(k)];
    if (out.size() != grid.node_count()) throw std::invalid_argument("hamiltonian: output size does not match the grid");
    if (dim < 0) {
        std::vector<const double*> cs;
        for (const ScalarField& c : costate) cs.push_back(c.values().data());
        check(lsg_eval_hamiltonian(ctx(), &g, &p, 0.0, cs.data(), out.values().data()));
    } else {
        check(lsg_eval_dissipation(ctx(), &g, &p, 0.0, dim, out.values().data()));
    }
}

void attach_device_plugins(HamiltonianProblem& problem) {
    const DeviceHamiltonian dev = problem.device;
    problem.ham_func = [dev](double, const Grid& grid, std::span<const ScalarField> costate, ScalarField& out) {
        if (costate.size() != static_cast<std::size_t>(grid.dim()))
            throw std::invalid_argument("hamiltonian: needs one costate field per dimension");
        device_eval(grid, dev, -1, costate, out);
    };
    problem.dissipation_bounds = [dev](double, const Grid& grid, int dim, ScalarField& out) {
        if (dim < 0 || dim >= grid.dim()) throw std::invalid_argument("dissipation: dimension out of range");
        device_eval(grid, dev, dim, {}, out);
    };
}

}  // namespace

void set_device(int device) { t_device = device; }

namespace detail {
void fill_padded_line(std::span<const double> field, std::size_t base, std::size_t stride, int n, int width,
                      BoundaryCondition bc, std::span<double> dst) {
    std::vector<double> line(static_cast<std::size_t>(n));
    for (int j = 0; j < n; ++j) line[static_cast<std::size_t>(j)] = field[base + static_cast<std::size_t>(j) * stride];
    lsg_grid g{};
    g.dim = 1;
    g.counts[0] = n;
    g.mins[0] = 0.0;
    g.maxs[0] = 1.0;
    g.periodic_mask = bc == BoundaryCondition::Periodic ? 1u : 0u;
    check(lsg_pad_ghost(ctx(), &g, line.data(), 0, width, dst.data()));
}
}  // namespace detail

// ---- Grid (grid.cpp:9-91) ---------------------------------------------------------
std::shared_ptr<const Grid> Grid::create(std::vector<double> mins, std::vector<double> maxs, std::vector<int> counts,
                                         const std::set<int>& periodic_dims) {
    const std::size_t dim = counts.size();
    if (dim == 0) throw std::invalid_argument("grid: dimension must be at least 1");
    if (mins.size() != dim || maxs.size() != dim)
        throw std::invalid_argument("grid: mins, maxs and counts must have equal length");
    for (std::size_t d = 0; d < dim; ++d) {
        if (counts[d] < 3) throw std::invalid_argument("grid: counts[" + std::to_string(d) + "] must be >= 3");
        if (!(maxs[d] > mins[d]))
            throw std::invalid_argument("grid: max must exceed min in dimension " + std::to_string(d));
    }
    for (int d : periodic_dims)
        if (d < 0 || d >= static_cast<int>(dim))
            throw std::invalid_argument("grid: periodic dimension " + std::to_string(d) + " out of range");
    auto g = std::shared_ptr<Grid>(new Grid());
    g->mins_ = std::move(mins);
    g->maxs_ = std::move(maxs);
    g->counts_ = std::move(counts);
    g->spacings_.resize(dim);
    g->boundary_.assign(dim, BoundaryCondition::ExtrapolateLinear);
    g->strides_.resize(dim);
    g->axes_.resize(dim);
    g->coord_fields_.resize(dim);
    std::size_t total = 1;
    for (std::size_t d = 0; d < dim; ++d) {
        const int n = g->counts_[d];
        g->spacings_[d] = (g->maxs_[d] - g->mins_[d]) / static_cast<double>(n - 1);
        if (periodic_dims.count(static_cast<int>(d))) g->boundary_[d] = BoundaryCondition::Periodic;
        g->strides_[d] = total;
        total *= static_cast<std::size_t>(n);
        g->axes_[d].resize(static_cast<std::size_t>(n));
        for (int i = 0; i < n; ++i)
            g->axes_[d][static_cast<std::size_t>(i)] = g->mins_[d] + static_cast<double>(i) * g->spacings_[d];
    }
    g->node_count_ = total;
    return g;
}

std::span<const double> Grid::coords(int d) const {
    auto& xs = coord_fields_[static_cast<std::size_t>(d)];
    if (xs.empty()) {
        xs.resize(node_count_);
        const auto& ax = axes_[static_cast<std::size_t>(d)];
        const std::size_t st = strides_[static_cast<std::size_t>(d)];
        const std::size_t block = st * static_cast<std::size_t>(counts_[static_cast<std::size_t>(d)]);
        for (std::size_t i = 0; i < node_count_; ++i) xs[i] = ax[(i % block) / st];
    }
    return xs;
}

std::size_t Grid::index(std::span<const int> multi) const {
    if (multi.size() != counts_.size()) throw std::invalid_argument("grid: multi-index length mismatch");
    std::size_t linear = 0;
    for (std::size_t d = 0; d < counts_.size(); ++d) {
        const int i = multi[d];
        if (i < 0 || i >= counts_[d]) throw std::out_of_range("grid: index out of range in dimension " + std::to_string(d));
        linear += static_cast<std::size_t>(i) * strides_[d];
    }
    return linear;
}

std::vector<int> Grid::multi_index(std::size_t linear) const {
    if (linear >= node_count_) throw std::out_of_range("grid: linear index out of range");
    std::vector<int> m(counts_.size());
    for (std::size_t d = 0; d < counts_.size(); ++d)
        m[d] = static_cast<int>((linear / strides_[d]) % static_cast<std::size_t>(counts_[d]));
    return m;
}

ScalarField::ScalarField(GridPtr grid, double fill) : grid_(std::move(grid)) {
    if (!grid_) throw std::invalid_argument("field: null grid");
    data_.assign(grid_->node_count(), fill);
}

ScalarField::ScalarField(GridPtr grid, std::vector<double> data) : grid_(std::move(grid)), data_(std::move(data)) {
    if (!grid_) throw std::invalid_argument("field: null grid");
    if (data_.size() != grid_->node_count())
        throw std::invalid_argument("field: data size does not match grid node count");
}

PaddedField pad_ghost(const ScalarField& field, int dim, int width) {
    const Grid& g = field.grid();
    lsg_grid c = to_c(g);
    PaddedField out;
    out.grid = field.grid_ptr();
    out.dim = dim;
    out.width = width;
    if (dim >= 0 && dim < g.dim() && width >= 1 && width < g.count(dim))
        out.data.resize(g.node_count() / static_cast<std::size_t>(g.count(dim)) *
                        static_cast<std::size_t>(g.count(dim) + 2 * width));
    check(lsg_pad_ghost(ctx(), &c, field.values().data(), dim, width, out.data.data()));
    return out;
}

ScalarField shift_along_dim(const PaddedField& padded, int offset) {
    if (!padded.grid) throw std::invalid_argument("shift_along_dim: padded field has no grid");
    lsg_grid c = to_c(*padded.grid);
    ScalarField out(padded.grid);
    check(lsg_shift_along_dim(ctx(), &c, padded.data.data(), padded.dim, padded.width, offset, out.values().data()));
    return out;
}

// ---- spatial_derivatives (spatial_derivatives.cpp:10-224) ----------------------------
int ghost_width(DerivativeScheme scheme) {
    switch (scheme) {
        case DerivativeScheme::First: return 1;
        case DerivativeScheme::Eno2: return 2;
        case DerivativeScheme::Eno3: return 3;
        case DerivativeScheme::Weno5: return 3;
    }
    throw std::invalid_argument("unknown derivative scheme");
}

int min_nodes(DerivativeScheme scheme) {
    switch (scheme) {
        case DerivativeScheme::First: return 3;
        case DerivativeScheme::Eno2: return 5;
        case DerivativeScheme::Eno3: return 7;
        case DerivativeScheme::Weno5: return 7;
    }
    throw std::invalid_argument("unknown derivative scheme");
}

DerivativePair upwind_derivative(const ScalarField& v, int dim, DerivativeScheme scheme) {
    lsg_grid c = to_c(v.grid());
    DerivativePair out{ScalarField(v.grid_ptr()), ScalarField(v.grid_ptr()), dim};
    check(lsg_upwind(ctx(), &c, v.values().data(), dim, scheme_c(scheme), out.left.values().data(),
                     out.right.values().data()));
    return out;
}

DerivativePair upwind_first_first(const ScalarField& v, int dim) { return upwind_derivative(v, dim, DerivativeScheme::First); }
DerivativePair upwind_first_eno2(const ScalarField& v, int dim) { return upwind_derivative(v, dim, DerivativeScheme::Eno2); }
DerivativePair upwind_first_eno3(const ScalarField& v, int dim) { return upwind_derivative(v, dim, DerivativeScheme::Eno3); }
DerivativePair upwind_first_weno5(const ScalarField& v, int dim) { return upwind_derivative(v, dim, DerivativeScheme::Weno5); }

// ---- Hamiltonian descriptors ----------------------------------------------------------
DeviceHamiltonian linear_hamiltonian(std::vector<double> c, std::vector<double> bounds, double offset) {
    if (c.size() > 6) throw std::invalid_argument("linear_hamiltonian: at most 6 dimensions");
    DeviceHamiltonian h;
    h.kind = LSG_HAM_LINEAR;
    for (std::size_t d = 0; d < c.size(); ++d) {
        h.params[d] = c[d];
        h.params[6 + d] = bounds.empty() ? std::abs(c[d]) : bounds.at(d);
    }
    h.params[12] = offset;
    return h;
}

DeviceHamiltonian air3d_hamiltonian(double v_a, double v_b, double w_a, double w_b) {
    DeviceHamiltonian h;
    h.kind = LSG_HAM_AIR3D;
    h.params[0] = v_a, h.params[1] = v_b, h.params[2] = w_a, h.params[3] = w_b;
    return h;
}

DeviceHamiltonian double_integrator4_hamiltonian() {
    DeviceHamiltonian h;
    h.kind = LSG_HAM_DBLINT4;
    return h;
}

DeviceHamiltonian dubins6_hamiltonian() {
    DeviceHamiltonian h;
    h.kind = LSG_HAM_DUBINS6;
    return h;
}

DeviceHamiltonian normal_motion_hamiltonian(double speed) {
    DeviceHamiltonian h;
    h.kind = LSG_HAM_NORMAL;
    h.params[0] = speed;
    return h;
}

// ---- hamiltonian.cpp:11-88 --------------------------------------------------------------
TermResult term_lax_friedrichs(double t, const ScalarField& v, const HamiltonianProblem& problem) {
    if (!problem.grid) throw std::invalid_argument("term_lax_friedrichs: problem has no grid");
    if (v.grid_ptr() != problem.grid)
        throw std::invalid_argument("term_lax_friedrichs: field grid does not match problem grid");
    lsg_grid g = to_c(*problem.grid);
    lsg_problem p = to_c(problem);
    TermResult r{ScalarField(problem.grid), 0.0};
    check(lsg_term_lf(ctx(), &g, &p, t, v.values().data(), r.dvdt.values().data(), &r.step_bound));
    return r;
}

ScalarField restrict_update(const ScalarField& dvdt, UpdateDirection direction) {
    ScalarField out(dvdt.grid_ptr());
    check(lsg_restrict_update(ctx(), dvdt.size(), dvdt.values().data(),
                              direction == UpdateDirection::Shrink ? LSG_SHRINK : LSG_GROW, out.values().data()));
    return out;
}

// ---- integrator.cpp:22-125 ---------------------------------------------------------------
TermFn make_lax_friedrichs_term(const HamiltonianProblem& problem) {
    return LaxFriedrichsTerm{std::make_shared<const HamiltonianProblem>(problem)};
}

IntegrationResult integrate(TimeIntegrator method, const TermFn& term, std::pair<double, double> tspan,
                            ScalarField v0, const IntegratorOptions& opts) {
    const LaxFriedrichsTerm* lf = term.target<LaxFriedrichsTerm>();
    if (!lf)
        throw std::invalid_argument(
            "integrate: the B200 path fuses the Lax-Friedrichs term into its RK stages; build the TermFn with "
            "make_lax_friedrichs_term (arbitrary host TermFns have no device path)");
    const HamiltonianProblem& problem = *lf->problem;
    if (v0.grid_ptr() != problem.grid)
        throw std::invalid_argument("term_lax_friedrichs: field grid does not match problem grid");
    lsg_grid g = to_c(*problem.grid);
    lsg_problem p = to_c(problem);
    OptsC o(opts);
    IntegrationResult r{tspan.first, std::move(v0), {}};
    std::vector<lsg_steplog> log(4096);
    std::size_t n = 0;
    double tfin = tspan.first;
    int rc = lsg_integrate(ctx(), &g, &p, static_cast<int>(method), tspan.first, tspan.second, r.v.values().data(),
                           &o.o, log.data(), log.size(), &n, &tfin);
    if (rc == LSG_ERANGE && n > log.size()) {  // the leg needs a longer log: nothing ran, retry
        log.resize(n);
        rc = lsg_integrate(ctx(), &g, &p, static_cast<int>(method), tspan.first, tspan.second, r.v.values().data(),
                           &o.o, log.data(), log.size(), &n, &tfin);
    }
    check(rc);
    r.t = tfin;
    r.steps = to_steps(log, n);
    return r;
}

IntegrationResult ode_cfl_1(const TermFn& term, std::pair<double, double> tspan, ScalarField v0,
                            const IntegratorOptions& opts) {
    return integrate(TimeIntegrator::Cfl1, term, tspan, std::move(v0), opts);
}
IntegrationResult ode_cfl_2(const TermFn& term, std::pair<double, double> tspan, ScalarField v0,
                            const IntegratorOptions& opts) {
    return integrate(TimeIntegrator::Cfl2, term, tspan, std::move(v0), opts);
}
IntegrationResult ode_cfl_3(const TermFn& term, std::pair<double, double> tspan, ScalarField v0,
                            const IntegratorOptions& opts) {
    return integrate(TimeIntegrator::Cfl3, term, tspan, std::move(v0), opts);
}

// ---- reachability.cpp:12-174 ---------------------------------------------------------------
double rocket_hamiltonian_value(double x, double theta, double p1, double p2, double p3, const RocketParams& params) {
    return -params.a * p1 * std::cos(theta) - p2 * (params.g - params.a - params.a * std::sin(theta)) -
           params.u_max * std::abs(p1 * x + p3) + params.u_min * std::abs(p2 * x + p3);
}

namespace {
DeviceHamiltonian rocket_device(const RocketParams& params) {
    DeviceHamiltonian d;
    d.kind = LSG_HAM_ROCKETS;
    d.params[0] = params.a;
    d.params[1] = params.g;
    d.params[2] = params.capture_radius;
    d.params[3] = params.u_min;
    d.params[4] = params.u_max;
    return d;
}
}  // namespace

void rocket_hamiltonian(double t, const Grid& grid, std::span<const ScalarField> costate, ScalarField& out,
                        const RocketParams& params) {
    (void)t;
    if (grid.dim() != 3) throw std::invalid_argument("rocket_hamiltonian: grid must be 3-D (x, z, theta)");
    if (costate.size() != 3) throw std::invalid_argument("rocket_hamiltonian: needs three costate fields");
    device_eval(grid, rocket_device(params), -1, costate, out);
}

void rocket_dissipation(double t, const Grid& grid, int dim, ScalarField& out, const RocketParams& params) {
    (void)t;
    if (grid.dim() != 3) throw std::invalid_argument("rocket_dissipation: grid must be 3-D (x, z, theta)");
    if (dim < 0 || dim > 2) throw std::invalid_argument("rocket_dissipation: dimension out of range");
    device_eval(grid, rocket_device(params), dim, {}, out);
}

ProblemSetup build_rocket_problem(int points_per_dim, const RocketParams& params, bool theta_periodic) {
    if (points_per_dim < 7) throw std::invalid_argument("build_rocket_problem: needs at least 7 points per dimension");
    if (!(params.u_max > params.u_min)) throw std::invalid_argument("build_rocket_problem: u_max must exceed u_min");
    if (!(params.capture_radius > 0.0))
        throw std::invalid_argument("build_rocket_problem: capture_radius must be positive");
    GridPtr grid;
    if (theta_periodic) {
        const double half_pi = 3.14159265358979323846 / 2.0;
        const double dtheta = 3.14159265358979323846 / static_cast<double>(points_per_dim);
        grid = Grid::create({-64.0, -64.0, -half_pi}, {64.0, 64.0, half_pi - dtheta},
                            {points_per_dim, points_per_dim, points_per_dim}, {2});
    } else {
        grid = Grid::create({-64.0, -64.0, -64.0}, {64.0, 64.0, 64.0}, {points_per_dim, points_per_dim, points_per_dim});
    }
    HamiltonianProblem problem;
    problem.grid = grid;
    problem.costate_scheme = DerivativeScheme::Eno2;
    problem.update_direction = UpdateDirection::Grow;
    problem.restrict_update = true;
    problem.device.kind = LSG_HAM_ROCKETS;
    problem.device.params[0] = params.a;
    problem.device.params[1] = params.g;
    problem.device.params[2] = params.capture_radius;
    problem.device.params[3] = params.u_min;
    problem.device.params[4] = params.u_max;
    attach_device_plugins(problem);
    ScalarField initial = cylinder(grid, {2}, {0.0, 0.0, 0.0}, params.capture_radius);
    return ProblemSetup{std::move(problem), std::move(initial)};
}

ProblemSetup rigid_rotation_problem(int points_per_dim) {
    if (points_per_dim < 7) throw std::invalid_argument("rigid_rotation_problem: needs at least 7 points per dimension");
    GridPtr grid = Grid::create({-1.0, -1.0}, {1.0, 1.0}, {points_per_dim, points_per_dim});
    HamiltonianProblem problem;
    problem.grid = grid;
    problem.costate_scheme = DerivativeScheme::Weno5;
    problem.update_direction = UpdateDirection::Grow;
    problem.restrict_update = false;
    problem.device.kind = LSG_HAM_ROTATION;
    attach_device_plugins(problem);
    ScalarField initial = sphere(grid, {0.5, 0.0}, 0.5);
    return ProblemSetup{std::move(problem), std::move(initial)};
}

SolveOutcome solve_brt(const ProblemSetup& setup, std::pair<double, double> tspan, int n_checkpoints,
                       TimeIntegrator method, const IntegratorOptions& opts) {
    if (setup.initial_value.grid_ptr() != setup.problem.grid)
        throw std::invalid_argument("solve_brt: initial value grid does not match problem grid");
    const GridPtr& grid = setup.problem.grid;
    lsg_grid g = to_c(*grid);
    SolveOutcome out;
    if (n_checkpoints < 1) throw std::invalid_argument("solve_brt: need at least one checkpoint");
    lsg_problem p{};
    const double duration = std::abs(tspan.second - tspan.first);
    if (std::isfinite(tspan.first) && std::isfinite(tspan.second) && duration != 0.0 && n_checkpoints > 1)
        p = to_c(setup.problem);
    const std::size_t N = grid->node_count();
    std::vector<double> ck(N * static_cast<std::size_t>(n_checkpoints));
    std::vector<double> times(static_cast<std::size_t>(n_checkpoints));
    std::vector<lsg_steplog> log(4096);
    int n_out = 0;
    std::size_t n_steps = 0;
    double seconds = 0.0;
    OptsC o(opts);
    auto call = [&] {
        return lsg_solve_brt(ctx(), &g, &p, setup.initial_value.values().data(), tspan.first, tspan.second,
                             n_checkpoints, static_cast<int>(method), &o.o, ck.data(), times.data(), &n_out,
                             log.data(), log.size(), &n_steps, &seconds);
    };
    int rc = call();
    if (rc == LSG_ERANGE && n_steps > log.size()) {  // nothing ran: retry with room for every step
        log.resize(n_steps);
        rc = call();
    }
    check(rc);
    for (int k = 0; k < n_out; ++k) {
        out.checkpoints.emplace_back(grid, std::vector<double>(ck.begin() + static_cast<std::ptrdiff_t>(k * N),
                                                                ck.begin() + static_cast<std::ptrdiff_t>((k + 1) * N)));
        out.checkpoint_times.push_back(times[static_cast<std::size_t>(k)]);
    }
    out.steps = to_steps(log, std::min(n_steps, log.size()));
    out.integration_seconds = seconds;
    return out;
}

// ---- runner.cpp:298-341 ---------------------------------------------------------------------
// runner.cpp:343-359, same stream formatting (host presentation of the device study)
std::string format_convergence_table(const std::vector<ConvergenceRow>& rows) {
    std::ostringstream os;
    os << std::setprecision(12);
    os << "n,dx,max_error,order\n";
    for (std::size_t i = 0; i < rows.size(); ++i) {
        const ConvergenceRow& row = rows[i];
        os << row.n << "," << row.dx << "," << row.max_error << ",";
        if (i == 0)
            os << "";
        else if (row.exact && rows[i - 1].exact)
            os << "exact";
        else
            os << row.order;
        os << "\n";
    }
    return os.str();
}

std::vector<ConvergenceRow> convergence_study(DerivativeScheme scheme, int refinements, const std::string& profile) {
    if (refinements < 1) throw std::invalid_argument("convergence_study: refinements must be at least 1");
    if (profile != "sin" && profile != "linear")
        throw std::invalid_argument("convergence_study: unknown profile '" + profile + "' (valid: sin, linear)");
    const bool periodic = profile == "sin";
    constexpr double two_pi = 2.0 * std::numbers::pi;
    std::vector<ConvergenceRow> rows;
    for (int level = 0; level <= refinements; ++level) {
        const int n = 32 << level;
        GridPtr grid = periodic ? Grid::create({0.0}, {1.0 - 1.0 / static_cast<double>(n)}, {n}, {0})
                                : Grid::create({0.0}, {1.0}, {n});
        ScalarField v(grid);
        for (int i = 0; i < n; ++i) {
            const double x = grid->axis(0)[static_cast<std::size_t>(i)];
            v[static_cast<std::size_t>(i)] = periodic ? std::sin(two_pi * x) : x;
        }
        const DerivativePair pair = upwind_derivative(v, 0, scheme);  // device
        double max_error = 0.0;
        for (int i = 0; i < n; ++i) {
            const double x = grid->axis(0)[static_cast<std::size_t>(i)];
            const double truth = periodic ? two_pi * std::cos(two_pi * x) : 1.0;
            max_error = std::max(max_error, std::abs(pair.left[static_cast<std::size_t>(i)] - truth));
            max_error = std::max(max_error, std::abs(pair.right[static_cast<std::size_t>(i)] - truth));
        }
        ConvergenceRow row;
        row.n = n;
        row.dx = grid->spacing(0);
        row.max_error = max_error;
        row.exact = max_error <= 1e-12;
        row.order = rows.empty() ? std::numeric_limits<double>::quiet_NaN() : std::log2(rows.back().max_error / max_error);
        rows.push_back(row);
    }
    return rows;
}

// ---- contour.cpp:27-142 -----------------------------------------------------------------------
std::vector<Segment2> extract_zero_set_2d(const ScalarField& field) {
    lsg_grid g = to_c(field.grid());
    std::vector<double> seg(4 * 4096);
    std::size_t n = 0;
    int rc = lsg_extract_zero_set_2d(ctx(), &g, field.values().data(), seg.data(), seg.size() / 4, &n);
    if (rc == LSG_ERANGE && n > seg.size() / 4) {
        seg.resize(4 * n);
        rc = lsg_extract_zero_set_2d(ctx(), &g, field.values().data(), seg.data(), n, &n);
    }
    check(rc);
    std::vector<Segment2> out(n);
    for (std::size_t k = 0; k < n; ++k) out[k] = {{seg[4 * k], seg[4 * k + 1]}, {seg[4 * k + 2], seg[4 * k + 3]}};
    return out;
}

ScalarField slice_2d(const ScalarField& field, int fixed_dim, int index) {
    const Grid& g = field.grid();
    lsg_grid c = to_c(g);
    if (g.dim() < 3) throw std::invalid_argument("slice_2d: field must be at least 3-D");
    if (fixed_dim < 0 || fixed_dim >= g.dim()) throw std::invalid_argument("slice_2d: fixed dimension out of range");
    std::vector<double> mins, maxs;
    std::vector<int> counts;
    std::set<int> periodic;
    for (int d = 0; d < g.dim(); ++d) {
        if (d == fixed_dim) continue;
        if (g.boundary(d) == BoundaryCondition::Periodic) periodic.insert(static_cast<int>(counts.size()));
        mins.push_back(g.min(d));
        maxs.push_back(g.max(d));
        counts.push_back(g.count(d));
    }
    GridPtr sg = Grid::create(mins, maxs, counts, periodic);
    ScalarField out(sg);
    check(lsg_slice_2d(ctx(), &c, field.values().data(), fixed_dim, index, out.values().data()));
    return out;
}

double polyline_length(const std::vector<Segment2>& segments) {
    double length = 0.0;
    for (const auto& s : segments) length += std::hypot(s.b.x - s.a.x, s.b.y - s.a.y);
    return length;
}

// ---- snapshot.cpp:69-129 ----------------------------------------------------------------------
void write_snapshot(const std::string& path, const ScalarField& field, double time) {
    lsg_grid g = to_c(field.grid());
    check(lsg_write_snapshot(&g, field.values().data(), time, path.c_str()));
}

Snapshot read_snapshot(const std::string& path) {
    lsg_grid g{};
    double t = 0.0;
    check(lsg_read_snapshot(path.c_str(), &g, &t, nullptr, 0));
    std::vector<double> mins(g.mins, g.mins + g.dim), maxs(g.maxs, g.maxs + g.dim);
    std::vector<int> counts(g.counts, g.counts + g.dim);
    GridPtr grid = Grid::create(mins, maxs, counts);
    std::vector<double> data(grid->node_count());
    check(lsg_read_snapshot(path.c_str(), &g, &t, data.data(), data.size()));
    return Snapshot{grid, ScalarField(grid, std::move(data)), t};
}

// ---- implicit_surfaces.cpp:20-71 (device generator) ----------------------------------------
ScalarField sphere(GridPtr grid, const std::vector<double>& center, double radius) {
    if (!grid) throw std::invalid_argument("sphere: null grid");
    if (center.size() != static_cast<std::size_t>(grid->dim()))
        throw std::invalid_argument("sphere: center length must equal the grid dimension");
    if (!(radius > 0.0)) throw std::invalid_argument("sphere: radius must be positive");
    return device_shape(grid, 0, 0u, center, radius);
}

ScalarField cylinder(GridPtr grid, const std::set<int>& ignored_dims, const std::vector<double>& center,
                     double radius) {
    if (!grid) throw std::invalid_argument("cylinder: null grid");
    if (center.size() != static_cast<std::size_t>(grid->dim()))
        throw std::invalid_argument("cylinder: center length must equal the grid dimension");
    if (!(radius > 0.0)) throw std::invalid_argument("cylinder: radius must be positive");
    if (ignored_dims.empty()) throw std::invalid_argument("cylinder: ignored_dims must be nonempty");
    unsigned mask = 0;
    for (int d : ignored_dims) {
        if (d < 0 || d >= grid->dim())
            throw std::invalid_argument("cylinder: ignored dimension " + std::to_string(d) + " out of range");
        mask |= 1u << d;
    }
    if (static_cast<int>(ignored_dims.size()) >= grid->dim())
        throw std::invalid_argument("cylinder: at least one dimension must remain active");
    return device_shape(grid, 1, mask, center, radius);
}

// implicit_surfaces.cpp:73-151 (argument checks and messages as the reference's)
ScalarField rectangle(GridPtr grid, const std::vector<double>& lower, const std::vector<double>& upper) {
    if (!grid) throw std::invalid_argument("rectangle: null grid");
    const std::size_t dim = static_cast<std::size_t>(grid->dim());
    if (lower.size() != dim || upper.size() != dim)
        throw std::invalid_argument("rectangle: corner length must equal the grid dimension");
    for (std::size_t d = 0; d < dim; ++d)
        if (!(upper[d] > lower[d]))
            throw std::invalid_argument("rectangle: upper must exceed lower in dimension " + std::to_string(d));
    return device_shape(grid, 3, 0u, lower, 0.0, upper);
}

ScalarField ellipsoid(GridPtr grid, double radius) {
    if (!grid) throw std::invalid_argument("ellipsoid: null grid");
    if (grid->dim() != 2 && grid->dim() != 3)
        throw std::invalid_argument("ellipsoid: only 2-D and 3-D grids are supported");
    if (!(radius > 0.0)) throw std::invalid_argument("ellipsoid: radius must be positive");
    return device_shape(grid, 4, 0u, {}, radius);
}

namespace {
ScalarField device_set_op(int op, const ScalarField& a, const ScalarField* b, const char* what) {
    if (b && a.grid_ptr() != b->grid_ptr())
        throw std::invalid_argument(std::string(what) + ": operands must share a grid");
    ScalarField out(a.grid_ptr());
    check(lsg_set_op(ctx(), op, a.size(), a.values().data(), b ? b->values().data() : nullptr,
                     out.values().data()));
    return out;
}
}  // namespace

ScalarField set_union(const ScalarField& a, const ScalarField& b) { return device_set_op(1, a, &b, "set_union"); }
ScalarField set_intersection(const ScalarField& a, const ScalarField& b) {
    return device_set_op(2, a, &b, "set_intersection");
}
ScalarField set_complement(const ScalarField& a) { return device_set_op(3, a, nullptr, "set_complement"); }

}  // namespace levelset
