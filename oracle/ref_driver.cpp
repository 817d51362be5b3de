// oracle/ref_driver.cpp — TEST INFRASTRUCTURE ONLY (the checker, never the product).
//
// C-ABI driver around the UNMODIFIED reference library, compiled from the
// reference's own sources under /root/reference/proj/core/src by
// oracle/Makefile into oracle/_ref/libref_levelset.so.  Only tests/,
// __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference arm
// load it.
//
// Every Hamiltonian kind of include/lsg.h is plugged in through the
// reference's own plugin API (HamiltonianFn / DissipationFn,
// hamiltonian.hpp:18-25); the two problems the reference ships (rockets,
// rigid rotation) reuse the reference's own lambdas and functions
// (reachability.cpp:12-66, :105-133).  The builder-defined config
// Hamiltonians (Air3D, double integrator, Dubins, normal motion) are written
// here with an explicit operation order that the CUDA kernels replicate.

#include <chrono>
#include <cmath>
#include <cstring>
#include <set>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "levelset/contour.hpp"
#include "levelset/grid.hpp"
#include "levelset/hamiltonian.hpp"
#include "levelset/implicit_surfaces.hpp"
#include "levelset/integrator.hpp"
#include "levelset/reachability.hpp"
#include "levelset/runner.hpp"
#include "levelset/snapshot.hpp"
#include "levelset/spatial_derivatives.hpp"

#include "../include/lsg.h"

using namespace levelset;

namespace {

thread_local std::string g_err;

template <typename F>
int guarded(F&& f) {
    try {
        f();
        return LSG_OK;
    } catch (const std::invalid_argument& e) {
        g_err = e.what();
        return LSG_EINVAL;
    } catch (const std::out_of_range& e) {
        g_err = e.what();
        return LSG_ERANGE;
    } catch (const std::runtime_error& e) {
        g_err = e.what();
        return LSG_ENUMERIC;
    } catch (const std::exception& e) {
        g_err = e.what();
        return LSG_EINVAL;
    }
}

GridPtr make_grid(const lsg_grid* g) {
    std::vector<double> mins(g->mins, g->mins + g->dim), maxs(g->maxs, g->maxs + g->dim);
    std::vector<int> counts(g->counts, g->counts + g->dim);
    std::set<int> periodic;
    for (int d = 0; d < g->dim; ++d)
        if (g->periodic_mask & (1u << d))
            periodic.insert(d);
    return Grid::create(mins, maxs, counts, periodic);
}

DerivativeScheme scheme_of(int s) {
    switch (s) {
        case LSG_SCHEME_FIRST: return DerivativeScheme::First;
        case LSG_SCHEME_ENO2: return DerivativeScheme::Eno2;
        case LSG_SCHEME_ENO3: return DerivativeScheme::Eno3;
        case LSG_SCHEME_WENO5: return DerivativeScheme::Weno5;
    }
    throw std::invalid_argument("ref: unknown scheme");
}

TimeIntegrator method_of(int m) {
    switch (m) {
        case LSG_CFL1: return TimeIntegrator::Cfl1;
        case LSG_CFL2: return TimeIntegrator::Cfl2;
        case LSG_CFL3: return TimeIntegrator::Cfl3;
    }
    throw std::invalid_argument("ref: unknown integrator");
}

HamiltonianProblem make_problem(GridPtr grid, const lsg_problem* p) {
    HamiltonianProblem hp;
    hp.grid = grid;
    hp.costate_scheme = scheme_of(p->scheme);
    hp.update_direction = p->direction == LSG_SHRINK ? UpdateDirection::Shrink : UpdateDirection::Grow;
    hp.restrict_update = p->restrict_update != 0;
    const int D = grid->dim();
    std::vector<double> prm(p->params, p->params + LSG_MAX_PARAMS);

    switch (p->kind) {
        case LSG_HAM_LINEAR: {
            // test_hamiltonian.cpp:18-36 (advection_problem) + constant offset
            // (test_hamiltonian.cpp:148-158).
            hp.ham_func = [prm, D](double, const Grid&, std::span<const ScalarField> costate,
                                   ScalarField& out) {
                for (std::size_t i = 0; i < out.size(); ++i) {
                    double h = 0.0;
                    for (int d = 0; d < D; ++d)
                        h += prm[static_cast<std::size_t>(d)] * costate[static_cast<std::size_t>(d)][i];
                    out[i] = h + prm[12];
                }
            };
            hp.dissipation_bounds = [prm](double, const Grid&, int dim, ScalarField& out) {
                for (std::size_t i = 0; i < out.size(); ++i)
                    out[i] = prm[6 + static_cast<std::size_t>(dim)];
            };
            break;
        }
        case LSG_HAM_ROTATION: {
            if (D != 2) throw std::invalid_argument("ref: rotation needs a 2-D grid");
            // the reference's own lambdas (reachability.cpp:113-126)
            ProblemSetup rot = rigid_rotation_problem(7);
            hp.ham_func = rot.problem.ham_func;
            hp.dissipation_bounds = rot.problem.dissipation_bounds;
            break;
        }
        case LSG_HAM_ROCKETS: {
            if (D != 3) throw std::invalid_argument("ref: rockets needs a 3-D grid");
            RocketParams rp;
            rp.a = prm[0];
            rp.g = prm[1];
            rp.capture_radius = prm[2];
            rp.u_min = prm[3];
            rp.u_max = prm[4];
            // reference functions (reachability.cpp:19-66)
            hp.ham_func = [rp](double t, const Grid& g, std::span<const ScalarField> costate, ScalarField& out) {
                rocket_hamiltonian(t, g, costate, out, rp);
            };
            hp.dissipation_bounds = [rp](double t, const Grid& g, int dim, ScalarField& out) {
                rocket_dissipation(t, g, dim, out, rp);
            };
            break;
        }
        case LSG_HAM_AIR3D: {
            if (D != 3) throw std::invalid_argument("ref: air3d needs a 3-D grid");
            const double va = prm[0], vb = prm[1], wa = prm[2], wb = prm[3];
            hp.ham_func = [=](double, const Grid& g, std::span<const ScalarField> costate, ScalarField& out) {
                const auto xs = g.coords(0), ys = g.coords(1), ps = g.coords(2);
                for (std::size_t i = 0; i < out.size(); ++i) {
                    const double c = std::cos(ps[i]), s = std::sin(ps[i]);
                    const double p0 = costate[0][i], p1 = costate[1][i], p2 = costate[2][i];
                    const double drift = ((-va) * p0 + (vb * c) * p0) + (vb * s) * p1;
                    const double turn = wa * std::abs((ys[i] * p0 - xs[i] * p1) - p2);
                    out[i] = -((drift + turn) - wb * std::abs(p2));
                }
            };
            hp.dissipation_bounds = [=](double, const Grid& g, int dim, ScalarField& out) {
                const auto xs = g.coords(0), ys = g.coords(1), ps = g.coords(2);
                for (std::size_t i = 0; i < out.size(); ++i) {
                    if (dim == 0)
                        out[i] = std::abs(-va + vb * std::cos(ps[i])) + wa * std::abs(ys[i]);
                    else if (dim == 1)
                        out[i] = std::abs(vb * std::sin(ps[i])) + wa * std::abs(xs[i]);
                    else
                        out[i] = wa + wb;
                }
            };
            break;
        }
        case LSG_HAM_DBLINT4: {
            if (D != 4) throw std::invalid_argument("ref: dblint4 needs a 4-D grid");
            hp.ham_func = [](double, const Grid& g, std::span<const ScalarField> costate, ScalarField& out) {
                const auto x1 = g.coords(1), x3 = g.coords(3);
                for (std::size_t i = 0; i < out.size(); ++i)
                    out[i] = ((costate[0][i] * x1[i] + costate[2][i] * x3[i]) - std::abs(costate[1][i])) -
                             std::abs(costate[3][i]);
            };
            hp.dissipation_bounds = [](double, const Grid& g, int dim, ScalarField& out) {
                const auto x1 = g.coords(1), x3 = g.coords(3);
                for (std::size_t i = 0; i < out.size(); ++i)
                    out[i] = dim == 0 ? std::abs(x1[i]) : dim == 2 ? std::abs(x3[i]) : 1.0;
            };
            break;
        }
        case LSG_HAM_DUBINS6: {
            if (D != 6) throw std::invalid_argument("ref: dubins6 needs a 6-D grid");
            hp.ham_func = [](double, const Grid& g, std::span<const ScalarField> costate, ScalarField& out) {
                const auto ta = g.coords(2), tb = g.coords(5);
                for (std::size_t i = 0; i < out.size(); ++i) {
                    const double ca = std::cos(ta[i]), sa = std::sin(ta[i]);
                    const double cb = std::cos(tb[i]), sb = std::sin(tb[i]);
                    out[i] = ((((costate[0][i] * ca + costate[1][i] * sa) + costate[3][i] * cb) +
                               costate[4][i] * sb) - std::abs(costate[2][i])) + std::abs(costate[5][i]);
                }
            };
            hp.dissipation_bounds = [](double, const Grid&, int, ScalarField& out) {
                for (std::size_t i = 0; i < out.size(); ++i)
                    out[i] = 1.0;
            };
            break;
        }
        case LSG_HAM_NORMAL: {
            const double speed = prm[0];
            hp.ham_func = [speed, D](double, const Grid&, std::span<const ScalarField> costate, ScalarField& out) {
                for (std::size_t i = 0; i < out.size(); ++i) {
                    double r2 = 0.0;
                    for (int d = 0; d < D; ++d) {
                        const double q = costate[static_cast<std::size_t>(d)][i];
                        r2 += q * q;
                    }
                    out[i] = speed * std::sqrt(r2);
                }
            };
            hp.dissipation_bounds = [speed](double, const Grid&, int, ScalarField& out) {
                for (std::size_t i = 0; i < out.size(); ++i)
                    out[i] = speed;
            };
            break;
        }
        default:
            throw std::invalid_argument("ref: unknown hamiltonian kind");
    }
    return hp;
}

IntegratorOptions make_opts(const lsg_opts* o) {
    IntegratorOptions opts;
    if (o) {
        opts.cfl_factor = o->cfl_factor;
        opts.max_step = o->max_step;
        opts.termination_epsilon = o->termination_epsilon;
        if (o->checkpoint_times && o->n_checkpoint_times)
            opts.checkpoint_times.assign(o->checkpoint_times, o->checkpoint_times + o->n_checkpoint_times);
    }
    return opts;
}

void copy_log(const std::vector<StepLogEntry>& steps, lsg_steplog* out, std::size_t cap, std::size_t* n) {
    if (n) *n = steps.size();
    if (!out) return;
    for (std::size_t k = 0; k < steps.size() && k < cap; ++k)
        out[k] = {steps[k].t, steps[k].dt, steps[k].step_bound, steps[k].v_min, steps[k].v_max};
}

} // namespace

#pragma GCC visibility push(default)
extern "C" {

const char* ref_last_error(void) { return g_err.c_str(); }

int ref_grid_axis(const lsg_grid* g, int d, double* out) {
    return guarded([&] {
        GridPtr grid = make_grid(g);
        auto ax = grid->axis(d);
        std::memcpy(out, ax.data(), ax.size() * sizeof(double));
    });
}

int ref_pad_ghost(const lsg_grid* g, const double* field, int dim, int width, double* out) {
    return guarded([&] {
        GridPtr grid = make_grid(g);
        ScalarField f(grid, std::vector<double>(field, field + grid->node_count()));
        PaddedField p = pad_ghost(f, dim, width);
        std::memcpy(out, p.data.data(), p.data.size() * sizeof(double));
    });
}

int ref_shift_along_dim(const lsg_grid* g, const double* padded, int dim, int width, int offset, double* out) {
    return guarded([&] {
        GridPtr grid = make_grid(g);
        if (dim < 0 || dim >= grid->dim()) throw std::invalid_argument("ref: dim out of range");
        PaddedField p;
        p.grid = grid;
        p.dim = dim;
        p.width = width;
        const std::size_t n = static_cast<std::size_t>(grid->count(dim));
        p.data.assign(padded, padded + grid->node_count() / n * (n + 2 * static_cast<std::size_t>(width)));
        ScalarField s = shift_along_dim(p, offset);
        std::memcpy(out, s.values().data(), s.size() * sizeof(double));
    });
}

int ref_upwind(const lsg_grid* g, const double* v, int dim, int scheme, double* left, double* right) {
    return guarded([&] {
        GridPtr grid = make_grid(g);
        ScalarField f(grid, std::vector<double>(v, v + grid->node_count()));
        DerivativePair d = upwind_derivative(f, dim, scheme_of(scheme));
        std::memcpy(left, d.left.values().data(), f.size() * sizeof(double));
        std::memcpy(right, d.right.values().data(), f.size() * sizeof(double));
    });
}

int ref_term_lf(const lsg_grid* g, const lsg_problem* p, double t, const double* v, double* dvdt,
                double* step_bound) {
    return guarded([&] {
        GridPtr grid = make_grid(g);
        HamiltonianProblem hp = make_problem(grid, p);
        ScalarField f(grid, std::vector<double>(v, v + grid->node_count()));
        TermResult r = term_lax_friedrichs(t, f, hp);
        std::memcpy(dvdt, r.dvdt.values().data(), f.size() * sizeof(double));
        *step_bound = r.step_bound;
    });
}

int ref_restrict_update(std::size_t n, const double* dvdt, int direction, double* out) {
    return guarded([&] {
        GridPtr grid = Grid::create({0.0}, {1.0}, {static_cast<int>(n)});
        ScalarField f(grid, std::vector<double>(dvdt, dvdt + n));
        ScalarField r = restrict_update(f, direction == LSG_SHRINK ? UpdateDirection::Shrink : UpdateDirection::Grow);
        std::memcpy(out, r.values().data(), n * sizeof(double));
    });
}

int ref_integrate(const lsg_grid* g, const lsg_problem* p, int method, double t0, double tf, double* v,
                  const lsg_opts* o, lsg_steplog* steps, std::size_t cap, std::size_t* n_steps,
                  double* t_final) {
    return guarded([&] {
        GridPtr grid = make_grid(g);
        HamiltonianProblem hp = make_problem(grid, p);
        ScalarField f(grid, std::vector<double>(v, v + grid->node_count()));
        TermFn term = [&hp](double t, const ScalarField& u) { return term_lax_friedrichs(t, u, hp); };
        IntegrationResult r = integrate(method_of(method), term, {t0, tf}, f, make_opts(o));
        std::memcpy(v, r.v.values().data(), f.size() * sizeof(double));
        copy_log(r.steps, steps, cap, n_steps);
        if (t_final) *t_final = r.t;
    });
}

int ref_solve_brt(const lsg_grid* g, const lsg_problem* p, const double* v0, double t_first, double t_second,
                  int n_checkpoints, int method, const lsg_opts* o, double* checkpoints,
                  double* checkpoint_times, int* n_out, lsg_steplog* steps, std::size_t cap,
                  std::size_t* n_steps, double* seconds) {
    return guarded([&] {
        GridPtr grid = make_grid(g);
        ProblemSetup setup{make_problem(grid, p),
                           ScalarField(grid, std::vector<double>(v0, v0 + grid->node_count()))};
        SolveOutcome out = solve_brt(setup, {t_first, t_second}, n_checkpoints, method_of(method), make_opts(o));
        const std::size_t N = grid->node_count();
        for (std::size_t k = 0; k < out.checkpoints.size(); ++k) {
            if (checkpoints)
                std::memcpy(checkpoints + k * N, out.checkpoints[k].values().data(), N * sizeof(double));
            if (checkpoint_times) checkpoint_times[k] = out.checkpoint_times[k];
        }
        if (n_out) *n_out = static_cast<int>(out.checkpoints.size());
        copy_log(out.steps, steps, cap, n_steps);
        if (seconds) *seconds = out.integration_seconds;
    });
}

// The reference's own rockets setup end to end: build_rocket_problem +
// solve_brt (acceptance.cpp:381-419 uses N=50, (-2.5, 0), 11 checkpoints).
int ref_solve_rockets(int n, int theta_periodic, double t_first, double t_second, int n_checkpoints,
                      double* final_v, lsg_steplog* steps, std::size_t cap, std::size_t* n_steps) {
    return guarded([&] {
        ProblemSetup setup = build_rocket_problem(n, RocketParams{}, theta_periodic != 0);
        SolveOutcome out = solve_brt(setup, {t_first, t_second}, n_checkpoints);
        const ScalarField& last = out.checkpoints.back();
        std::memcpy(final_v, last.values().data(), last.size() * sizeof(double));
        copy_log(out.steps, steps, cap, n_steps);
    });
}

int ref_rocket_initial(int n, int theta_periodic, double* out) {
    return guarded([&] {
        ProblemSetup setup = build_rocket_problem(n, RocketParams{}, theta_periodic != 0);
        std::memcpy(out, setup.initial_value.values().data(), setup.initial_value.size() * sizeof(double));
    });
}

// implicit_surfaces.cpp:20-71
int ref_sphere(const lsg_grid* g, const double* center, double radius, double* out) {
    return guarded([&] {
        GridPtr grid = make_grid(g);
        ScalarField f = sphere(grid, std::vector<double>(center, center + grid->dim()), radius);
        std::memcpy(out, f.values().data(), f.size() * sizeof(double));
    });
}

int ref_cylinder(const lsg_grid* g, unsigned ignored_mask, const double* center, double radius, double* out) {
    return guarded([&] {
        GridPtr grid = make_grid(g);
        std::set<int> ignored;
        for (int d = 0; d < grid->dim(); ++d)
            if (ignored_mask & (1u << d)) ignored.insert(d);
        ScalarField f = cylinder(grid, ignored, std::vector<double>(center, center + grid->dim()), radius);
        std::memcpy(out, f.values().data(), f.size() * sizeof(double));
    });
}

// reachability.cpp:19-66: the rockets plugins on given costate fields
int ref_rocket_plugins(const lsg_grid* g, const double* params5, const double* p0, const double* p1,
                       const double* p2, double* h_out, double* b0, double* b1, double* b2) {
    return guarded([&] {
        GridPtr grid = make_grid(g);
        const std::size_t n = grid->node_count();
        RocketParams rp;
        rp.a = params5[0];
        rp.g = params5[1];
        rp.capture_radius = params5[2];
        rp.u_min = params5[3];
        rp.u_max = params5[4];
        std::vector<ScalarField> cs;
        for (const double* c : {p0, p1, p2}) cs.emplace_back(grid, std::vector<double>(c, c + n));
        ScalarField h(grid);
        rocket_hamiltonian(0.0, *grid, std::span<const ScalarField>(cs), h, rp);
        std::memcpy(h_out, h.values().data(), n * sizeof(double));
        double* bs[3] = {b0, b1, b2};
        for (int d = 0; d < 3; ++d) {
            ScalarField b(grid);
            rocket_dissipation(0.0, *grid, d, b, rp);
            std::memcpy(bs[d], b.values().data(), n * sizeof(double));
        }
    });
}

// implicit_surfaces.cpp:73-151
int ref_rectangle(const lsg_grid* g, const double* lower, const double* upper, double* out) {
    return guarded([&] {
        GridPtr grid = make_grid(g);
        ScalarField f = rectangle(grid, std::vector<double>(lower, lower + grid->dim()),
                                  std::vector<double>(upper, upper + grid->dim()));
        std::memcpy(out, f.values().data(), f.size() * sizeof(double));
    });
}

int ref_ellipsoid(const lsg_grid* g, double radius, double* out) {
    return guarded([&] {
        GridPtr grid = make_grid(g);
        ScalarField f = ellipsoid(grid, radius);
        std::memcpy(out, f.values().data(), f.size() * sizeof(double));
    });
}

// op 1 set_union, 2 set_intersection, 3 set_complement (b unused)
int ref_set_op(const lsg_grid* g, int op, const double* a, const double* b, double* out) {
    return guarded([&] {
        GridPtr grid = make_grid(g);
        const std::size_t n = grid->node_count();
        ScalarField fa(grid, std::vector<double>(a, a + n));
        ScalarField r = op == 3 ? set_complement(fa)
                                : (op == 1 ? set_union(fa, ScalarField(grid, std::vector<double>(b, b + n)))
                                           : set_intersection(fa, ScalarField(grid, std::vector<double>(b, b + n))));
        std::memcpy(out, r.values().data(), n * sizeof(double));
    });
}

// CPU baseline: `nthreads` concurrent independent replicas of the reference's
// integrate(method, LF term, {0, tf}, v0, opts) — the bench_kernels.cpp:70-83
// pattern, timed with steady_clock.  Returns wall seconds and the accepted
// step count of one replica.
int ref_bench(const lsg_grid* g, const lsg_problem* p, int method, const double* v0, double tf,
              const lsg_opts* o, int nthreads, double* seconds, std::size_t* steps_per_replica) {
    return guarded([&] {
        GridPtr grid = make_grid(g);
        HamiltonianProblem hp = make_problem(grid, p);
        const ScalarField f(grid, std::vector<double>(v0, v0 + grid->node_count()));
        const IntegratorOptions opts = make_opts(o);
        const TimeIntegrator m = method_of(method);
        std::vector<std::size_t> counts(static_cast<std::size_t>(nthreads), 0);
        std::vector<std::string> errs(static_cast<std::size_t>(nthreads));
        auto work = [&](int r) {
            try {
                TermFn term = [&hp](double t, const ScalarField& u) { return term_lax_friedrichs(t, u, hp); };
                IntegrationResult res = integrate(m, term, {0.0, tf}, f, opts);
                counts[static_cast<std::size_t>(r)] = res.steps.size();
            } catch (const std::exception& e) {
                errs[static_cast<std::size_t>(r)] = e.what();
            }
        };
        const auto start = std::chrono::steady_clock::now();
        std::vector<std::thread> pool;
        for (int r = 1; r < nthreads; ++r) pool.emplace_back(work, r);
        work(0);
        for (auto& th : pool) th.join();
        const auto stop = std::chrono::steady_clock::now();
        for (auto& e : errs)
            if (!e.empty()) throw std::runtime_error(e);
        *seconds = std::chrono::duration<double>(stop - start).count();
        *steps_per_replica = counts[0];
    });
}

// snapshot.cpp:69-129
int ref_write_snapshot(const lsg_grid* g, const double* field, double time, const char* path) {
    return guarded([&] {
        GridPtr grid = make_grid(g);
        write_snapshot(path, ScalarField(grid, std::vector<double>(field, field + grid->node_count())), time);
    });
}

int ref_read_snapshot(const char* path, lsg_grid* g, double* time, double* field, std::size_t cap) {
    return guarded([&] {
        Snapshot s = read_snapshot(path);
        lsg_grid out{};
        out.dim = s.grid->dim();
        for (int d = 0; d < out.dim && d < LSG_MAX_DIM; ++d) {
            out.counts[d] = s.grid->count(d);
            out.mins[d] = s.grid->min(d);
            out.maxs[d] = s.grid->max(d);
        }
        *g = out;
        *time = s.time;
        if (field) {
            if (cap < s.field.size()) throw std::invalid_argument("ref: buffer too small");
            std::memcpy(field, s.field.values().data(), s.field.size() * sizeof(double));
        }
    });
}

// contour.cpp:27-142
int ref_extract_zero_set_2d(const lsg_grid* g, const double* field, double* segs, std::size_t cap, std::size_t* n,
                            double* length) {
    return guarded([&] {
        GridPtr grid = make_grid(g);
        auto s = extract_zero_set_2d(ScalarField(grid, std::vector<double>(field, field + grid->node_count())));
        *n = s.size();
        for (std::size_t k = 0; k < s.size() && k < cap; ++k) {
            segs[4 * k] = s[k].a.x, segs[4 * k + 1] = s[k].a.y, segs[4 * k + 2] = s[k].b.x, segs[4 * k + 3] = s[k].b.y;
        }
        *length = polyline_length(s);
    });
}

int ref_slice_2d(const lsg_grid* g, const double* field, int fixed_dim, int index, double* out) {
    return guarded([&] {
        GridPtr grid = make_grid(g);
        ScalarField sl = slice_2d(ScalarField(grid, std::vector<double>(field, field + grid->node_count())), fixed_dim, index);
        std::memcpy(out, sl.values().data(), sl.size() * sizeof(double));
    });
}

// runner.cpp:298-341: rows of (n, dx, max_error, order)
int ref_convergence_study(int scheme, int refinements, int periodic, double* rows, int* nrows) {
    return guarded([&] {
        auto r = convergence_study(scheme_of(scheme), refinements, periodic ? "sin" : "linear");
        for (std::size_t k = 0; k < r.size(); ++k) {
            rows[4 * k + 0] = r[k].n;
            rows[4 * k + 1] = r[k].dx;
            rows[4 * k + 2] = r[k].max_error;
            rows[4 * k + 3] = r[k].order;
        }
        *nrows = static_cast<int>(r.size());
    });
}

} // extern "C"
#pragma GCC visibility pop
