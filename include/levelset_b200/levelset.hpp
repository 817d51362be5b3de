// levelset_b200/levelset.hpp — C++ drop-in for the reference library's hot path.
//
// Same namespace, type names, signatures and exception types as the
// reference headers (/root/reference/proj/core/include/levelset/):
//   grid.hpp               Grid, GridPtr, ScalarField, PaddedField, pad_ghost, shift_along_dim
//   spatial_derivatives.hpp DerivativeScheme, ghost_width, min_nodes, DerivativePair,
//                           upwind_first_first/eno2/eno3/weno5, upwind_derivative
//   hamiltonian.hpp        UpdateDirection, HamiltonianFn, DissipationFn, HamiltonianProblem,
//                           TermResult, term_lax_friedrichs, restrict_update
//   integrator.hpp         IntegratorOptions, StepLogEntry, IntegrationResult, TermFn,
//                           ode_cfl_1/2/3, TimeIntegrator, integrate
//   reachability.hpp       RocketParams, rocket_hamiltonian_value, ProblemSetup,
//                           build_rocket_problem, rigid_rotation_problem, SolveOutcome, solve_brt
//   implicit_surfaces.hpp  sphere, cylinder
// Every computation runs on the B200 through the C ABI (include/lsg.h); link
// liblevelset_b200.so instead of liblevelset.a.
//
// The one interface difference: the reference's Hamiltonian plugins are host
// std::function objects (hamiltonian.hpp:18-25) that a GPU cannot call, so a
// HamiltonianProblem also carries a DeviceHamiltonian (kind + POD params).
// The std::function members are kept for source compatibility but are never
// invoked; a problem without a device Hamiltonian, or an integrate() call with
// an arbitrary TermFn, throws std::invalid_argument — there is no CPU fallback.
#pragma once

#include <array>
#include <cstddef>
#include <functional>
#include <limits>
#include <memory>
#include <set>
#include <span>
#include <string>
#include <utility>
#include <vector>

namespace levelset {

// ---- grid.hpp ---------------------------------------------------------------
enum class BoundaryCondition { Periodic, ExtrapolateLinear };

class Grid {
public:
    static std::shared_ptr<const Grid> create(std::vector<double> mins, std::vector<double> maxs,
                                              std::vector<int> counts, const std::set<int>& periodic_dims = {});
    int dim() const { return static_cast<int>(counts_.size()); }
    double min(int d) const { return mins_[static_cast<std::size_t>(d)]; }
    double max(int d) const { return maxs_[static_cast<std::size_t>(d)]; }
    int count(int d) const { return counts_[static_cast<std::size_t>(d)]; }
    double spacing(int d) const { return spacings_[static_cast<std::size_t>(d)]; }
    BoundaryCondition boundary(int d) const { return boundary_[static_cast<std::size_t>(d)]; }
    std::size_t node_count() const { return node_count_; }
    std::size_t stride(int d) const { return strides_[static_cast<std::size_t>(d)]; }
    std::span<const double> axis(int d) const { return axes_[static_cast<std::size_t>(d)]; }
    /// Full coordinate field of dimension d, materialised on first use (host
    /// memory; not used by the device path, which indexes the axis tables).
    std::span<const double> coords(int d) const;
    std::size_t index(std::span<const int> multi) const;
    std::vector<int> multi_index(std::size_t linear) const;

private:
    Grid() = default;
    std::vector<double> mins_, maxs_, spacings_;
    std::vector<int> counts_;
    std::vector<BoundaryCondition> boundary_;
    std::vector<std::size_t> strides_;
    std::size_t node_count_ = 0;
    std::vector<std::vector<double>> axes_;
    mutable std::vector<std::vector<double>> coord_fields_;
};

using GridPtr = std::shared_ptr<const Grid>;

class ScalarField {
public:
    explicit ScalarField(GridPtr grid, double fill = 0.0);
    ScalarField(GridPtr grid, std::vector<double> data);
    const Grid& grid() const { return *grid_; }
    const GridPtr& grid_ptr() const { return grid_; }
    std::size_t size() const { return data_.size(); }
    double operator[](std::size_t i) const { return data_[i]; }
    double& operator[](std::size_t i) { return data_[i]; }
    std::span<const double> values() const { return data_; }
    std::span<double> values() { return data_; }
    double at(std::span<const int> multi) const { return data_[grid_->index(multi)]; }
    double& at(std::span<const int> multi) { return data_[grid_->index(multi)]; }

private:
    GridPtr grid_;
    std::vector<double> data_;
};

struct PaddedField {
    GridPtr grid;
    int dim = 0;
    int width = 0;
    std::vector<double> data;
};

PaddedField pad_ghost(const ScalarField& field, int dim, int width);

namespace detail {
/// grid.cpp:108-128: one line (n nodes at `base`, step `stride`) into
/// dst[width..width+n) plus `width` ghost nodes per side (ghost fill on the device).
void fill_padded_line(std::span<const double> field, std::size_t base, std::size_t stride, int n, int width,
                      BoundaryCondition bc, std::span<double> dst);
}  // namespace detail
ScalarField shift_along_dim(const PaddedField& padded, int offset);

// ---- spatial_derivatives.hpp -----------------------------------------------
enum class DerivativeScheme { First, Eno2, Eno3, Weno5 };
int ghost_width(DerivativeScheme scheme);
int min_nodes(DerivativeScheme scheme);

struct DerivativePair {
    ScalarField left;
    ScalarField right;
    int dim = 0;
};

DerivativePair upwind_first_first(const ScalarField& v, int dim);
DerivativePair upwind_first_eno2(const ScalarField& v, int dim);
DerivativePair upwind_first_eno3(const ScalarField& v, int dim);
DerivativePair upwind_first_weno5(const ScalarField& v, int dim);
DerivativePair upwind_derivative(const ScalarField& v, int dim, DerivativeScheme scheme);

// ---- hamiltonian.hpp ----------------------------------------------------------
enum class UpdateDirection { Grow, Shrink };

using HamiltonianFn =
    std::function<void(double t, const Grid& grid, std::span<const ScalarField> costate, ScalarField& out)>;
using DissipationFn = std::function<void(double t, const Grid& grid, int dim, ScalarField& out)>;

/// Device Hamiltonian: an LSG_HAM_* kind of include/lsg.h and its parameters.
struct DeviceHamiltonian {
    int kind = 0;  // 0: none
    std::array<double, 16> params{};
};

/// H = sum_d c_d p_d + offset, bounds b_d (test_hamiltonian.cpp:18-36 form).
DeviceHamiltonian linear_hamiltonian(std::vector<double> c, std::vector<double> bounds = {}, double offset = 0.0);
/// ToolboxLS air3D game (BASELINE cfg2).
DeviceHamiltonian air3d_hamiltonian(double v_a = 5.0, double v_b = 5.0, double w_a = 1.0, double w_b = 1.0);
DeviceHamiltonian double_integrator4_hamiltonian();
DeviceHamiltonian dubins6_hamiltonian();
DeviceHamiltonian normal_motion_hamiltonian(double speed = 1.0);

struct HamiltonianProblem {
    GridPtr grid;
    HamiltonianFn ham_func;              // device kinds: set to the device evaluator (callable like the
    DissipationFn dissipation_bounds;    // reference's plugins); the solver itself uses `device`, fused
    DerivativeScheme costate_scheme = DerivativeScheme::Eno2;
    UpdateDirection update_direction = UpdateDirection::Grow;
    bool restrict_update = false;
    DeviceHamiltonian device;            // what the B200 path evaluates
    unsigned options = 0;                // LSG_OPT_* (e.g. LSG_OPT_WENO5_FAST)
};

struct TermResult {
    ScalarField dvdt;
    double step_bound = 0.0;
};

TermResult term_lax_friedrichs(double t, const ScalarField& v, const HamiltonianProblem& problem);
ScalarField restrict_update(const ScalarField& dvdt, UpdateDirection direction);

// ---- integrator.hpp -------------------------------------------------------------
struct IntegratorOptions {
    double cfl_factor = 0.32;
    double max_step = std::numeric_limits<double>::infinity();
    double termination_epsilon = 1e-6;
    std::vector<double> checkpoint_times;
};

struct StepLogEntry {
    double t = 0.0;
    double dt = 0.0;
    double step_bound = 0.0;
    double v_min = 0.0;
    double v_max = 0.0;
};

struct IntegrationResult {
    double t = 0.0;
    ScalarField v;
    std::vector<StepLogEntry> steps;
};

using TermFn = std::function<TermResult(double t, const ScalarField& v)>;

/// The Lax-Friedrichs term as a recognisable TermFn target: integrate() runs
/// it fused on the device.  Call sites that wrap term_lax_friedrichs in a
/// lambda (reachability.cpp:154-156) use make_lax_friedrichs_term instead.
struct LaxFriedrichsTerm {
    std::shared_ptr<const HamiltonianProblem> problem;
    TermResult operator()(double t, const ScalarField& v) const { return term_lax_friedrichs(t, v, *problem); }
};
TermFn make_lax_friedrichs_term(const HamiltonianProblem& problem);

IntegrationResult ode_cfl_1(const TermFn& term, std::pair<double, double> tspan, ScalarField v0,
                            const IntegratorOptions& opts = {});
IntegrationResult ode_cfl_2(const TermFn& term, std::pair<double, double> tspan, ScalarField v0,
                            const IntegratorOptions& opts = {});
IntegrationResult ode_cfl_3(const TermFn& term, std::pair<double, double> tspan, ScalarField v0,
                            const IntegratorOptions& opts = {});

enum class TimeIntegrator { Cfl1, Cfl2, Cfl3 };

IntegrationResult integrate(TimeIntegrator method, const TermFn& term, std::pair<double, double> tspan,
                            ScalarField v0, const IntegratorOptions& opts = {});

// ---- reachability.hpp -------------------------------------------------------------
struct RocketParams {
    double a = 1.0;
    double g = 32.0;
    double capture_radius = 1.5;
    double u_min = -1.0;
    double u_max = 1.0;
};

double rocket_hamiltonian_value(double x, double theta, double p1, double p2, double p3, const RocketParams& params);
/// reachability.cpp:19-66 on the device (lsg_eval_hamiltonian / lsg_eval_dissipation).
void rocket_hamiltonian(double t, const Grid& grid, std::span<const ScalarField> costate, ScalarField& out,
                        const RocketParams& params);
void rocket_dissipation(double t, const Grid& grid, int dim, ScalarField& out, const RocketParams& params);

struct ProblemSetup {
    HamiltonianProblem problem;
    ScalarField initial_value;
};

ProblemSetup build_rocket_problem(int points_per_dim, const RocketParams& params = {}, bool theta_periodic = false);
ProblemSetup rigid_rotation_problem(int points_per_dim);

struct SolveOutcome {
    std::vector<ScalarField> checkpoints;
    std::vector<double> checkpoint_times;
    std::vector<StepLogEntry> steps;
    double integration_seconds = 0.0;
};

SolveOutcome solve_brt(const ProblemSetup& setup, std::pair<double, double> tspan, int n_checkpoints,
                       TimeIntegrator method = TimeIntegrator::Cfl3, const IntegratorOptions& opts = {});

// ---- implicit_surfaces.hpp (device initial-condition generator) -------------------
ScalarField sphere(GridPtr grid, const std::vector<double>& center, double radius);
ScalarField cylinder(GridPtr grid, const std::set<int>& ignored_dims, const std::vector<double>& center,
                     double radius);
ScalarField rectangle(GridPtr grid, const std::vector<double>& lower, const std::vector<double>& upper);
ScalarField ellipsoid(GridPtr grid, double radius);
ScalarField set_union(const ScalarField& a, const ScalarField& b);
ScalarField set_intersection(const ScalarField& a, const ScalarField& b);
ScalarField set_complement(const ScalarField& a);

// ---- runner.hpp: convergence study on the device kernels ---------------------------
struct ConvergenceRow {
    int n = 0;
    double dx = 0.0;
    double max_error = 0.0;
    double order = 0.0;  // NaN on the coarsest level
    bool exact = false;  // error at rounding level; order not meaningful
};
/// runner.cpp:298-341 with upwind_derivative on the B200 (profile "sin" or "linear").
std::vector<ConvergenceRow> convergence_study(DerivativeScheme scheme, int refinements,
                                              const std::string& profile = "sin");
/// runner.cpp:343-359: the study as CSV text (n,dx,max_error,order).
std::string format_convergence_table(const std::vector<ConvergenceRow>& rows);

// ---- contour.hpp: zero-level-set extraction on the device ----------------------------
struct Point2 {
    double x = 0.0;
    double y = 0.0;
};
struct Segment2 {
    Point2 a;
    Point2 b;
};
/// contour.cpp:27-97 — marching squares on the B200, same segments in the same order.
std::vector<Segment2> extract_zero_set_2d(const ScalarField& field);
/// contour.cpp:99-135 — 2-D slice of a 3-D field (device gather).
ScalarField slice_2d(const ScalarField& field, int fixed_dim, int index);
/// contour.cpp:137-142 — total length (host sum of std::hypot over the segments).
double polyline_length(const std::vector<Segment2>& segments);

// ---- snapshot.hpp: checkpoint files in the reference format --------------------------
struct Snapshot {
    GridPtr grid;
    ScalarField field;
    double time = 0.0;
};
void write_snapshot(const std::string& path, const ScalarField& field, double time);
Snapshot read_snapshot(const std::string& path);

// ---- device selection -----------------------------------------------------------------
/// CUDA device used by this thread's calls (default 0).
void set_device(int device);

}  // namespace levelset
