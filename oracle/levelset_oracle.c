/*
 * oracle/levelset_oracle.c — TEST INFRASTRUCTURE ONLY.
 *
 * Plain-C restatement of the reference hot path (/root/reference/proj/core,
 * paths below relative to it): ghost fill, upwind First/ENO2/ENO3/WENO5,
 * the Lax-Friedrichs term with global alpha and the update clamp, and the
 * CFL-controlled TVD-RK1/2/3 integrators plus the solve_brt leg driver.
 * It is the checker the CUDA path is compared against; only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline leg may load it.
 *
 * Parity pinning: tests/test_oracle.py checks this restatement bit-for-bit
 * against (1) the reference library itself, compiled from its own sources
 * into oracle/_ref/ by oracle/Makefile, and (2) the committed golden vectors
 * under tests/golden/ (made by tests/golden/make_golden.py from that build)
 * plus the reference's own known-answer tests.
 *
 * Compiled with -ffp-contract=off: IEEE fp64, round-to-nearest, no FMA, and
 * every expression keeps the reference's C++ evaluation order.
 */
#include <math.h>
#include <stdarg.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "../include/lsg.h"

static char orc_err[512];

static int fail(int code, const char* fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(orc_err, sizeof orc_err, fmt, ap);
    va_end(ap);
    return code;
}

const char* orc_last_error(void) { return orc_err; }

/* std::min / std::max as libstdc++ defines them: min(a,b) = (b < a) ? b : a. */
static double smin(double a, double b) { return (b < a) ? b : a; }
static double smax(double a, double b) { return (a < b) ? b : a; }

/* ---- grid (grid.cpp:9-66) ---------------------------------------------- */

int orc_grid_check(const lsg_grid* g) {
    if (!g || g->dim <= 0) return fail(LSG_EINVAL, "grid: dimension must be at least 1");
    if (g->dim > LSG_MAX_DIM) return fail(LSG_EINVAL, "grid: at most %d dimensions", LSG_MAX_DIM);
    for (int d = 0; d < g->dim; ++d) {
        if (g->counts[d] < 3) return fail(LSG_EINVAL, "grid: counts[%d] must be >= 3", d);
        if (!(g->maxs[d] > g->mins[d])) return fail(LSG_EINVAL, "grid: max must exceed min in dimension %d", d);
    }
    if (g->periodic_mask >> g->dim) return fail(LSG_EINVAL, "grid: periodic dimension out of range");
    return LSG_OK;
}

/* grid.cpp:41 */
double orc_spacing(const lsg_grid* g, int d) {
    return (g->maxs[d] - g->mins[d]) / (double)(g->counts[d] - 1);
}

size_t orc_node_count(const lsg_grid* g) {
    size_t n = 1;
    for (int d = 0; d < g->dim; ++d) n *= (size_t)g->counts[d];
    return n;
}

static size_t stride_of(const lsg_grid* g, int d) {
    size_t s = 1;
    for (int k = 0; k < d; ++k) s *= (size_t)g->counts[k];
    return s;
}

/* grid.cpp:50  axis[i] = min + i * dx */
void orc_axis(const lsg_grid* g, int d, double* out) {
    const double dx = orc_spacing(g, d);
    for (int i = 0; i < g->counts[d]; ++i) out[i] = g->mins[d] + (double)i * dx;
}

static int bc_of(const lsg_grid* g, int d) {
    return (g->periodic_mask >> d) & 1u ? LSG_BC_PERIODIC : LSG_BC_EXTRAPOLATE;
}

/* ---- ghost fill (grid.cpp:108-128) ------------------------------------ */

void orc_fill_padded_line(const double* field, size_t base, size_t stride, int n, int width, int bc,
                          double* dst) {
    for (int j = 0; j < n; ++j) dst[width + j] = field[base + (size_t)j * stride];
    if (bc == LSG_BC_PERIODIC) {
        for (int k = 0; k < width; ++k) {
            dst[k] = dst[k + n];
            dst[width + n + k] = dst[width + k];
        }
    } else {
        const double lo = dst[width];
        const double lo_slope = lo - dst[width + 1];
        const double hi = dst[width + n - 1];
        const double hi_slope = hi - dst[width + n - 2];
        for (int k = 1; k <= width; ++k) {
            dst[width - k] = lo + (double)k * lo_slope;
            dst[width + n - 1 + k] = hi + (double)k * hi_slope;
        }
    }
}

/* grid.cpp:132-165 */
int orc_pad_ghost(const lsg_grid* g, const double* field, int dim, int width, double* out) {
    int rc = orc_grid_check(g);
    if (rc) return rc;
    if (dim < 0 || dim >= g->dim) return fail(LSG_EINVAL, "pad_ghost: dimension out of range");
    if (width < 1) return fail(LSG_EINVAL, "pad_ghost: width must be >= 1");
    const int n = g->counts[dim];
    if (width >= n) return fail(LSG_EINVAL, "pad_ghost: width must be smaller than the node count along dim");
    const size_t stride = stride_of(g, dim);
    const size_t line_block = stride * (size_t)n;
    const size_t padded_block = stride * (size_t)(n + 2 * width);
    const size_t n_outer = orc_node_count(g) / line_block;
    double* s = (double*)malloc(sizeof(double) * (size_t)(n + 2 * width));
    for (size_t outer = 0; outer < n_outer; ++outer)
        for (size_t inner = 0; inner < stride; ++inner) {
            orc_fill_padded_line(field, outer * line_block + inner, stride, n, width, bc_of(g, dim), s);
            for (int j = 0; j < n + 2 * width; ++j) out[outer * padded_block + inner + (size_t)j * stride] = s[j];
        }
    free(s);
    return LSG_OK;
}

/* grid.cpp:167-193 */
int orc_shift_along_dim(const lsg_grid* g, const double* padded, int dim, int width, int offset, double* out) {
    int rc = orc_grid_check(g);
    if (rc) return rc;
    if (dim < 0 || dim >= g->dim) return fail(LSG_EINVAL, "shift_along_dim: dimension out of range");
    if (offset < -width || offset > width)
        return fail(LSG_EINVAL, "shift_along_dim: |offset| must not exceed the ghost width");
    const int n = g->counts[dim];
    const size_t stride = stride_of(g, dim);
    const size_t line_block = stride * (size_t)n;
    const size_t padded_block = stride * (size_t)(n + 2 * width);
    const size_t n_outer = orc_node_count(g) / line_block;
    const int start = width + offset;
    for (size_t outer = 0; outer < n_outer; ++outer)
        for (size_t inner = 0; inner < stride; ++inner)
            for (int j = 0; j < n; ++j)
                out[outer * line_block + inner + (size_t)j * stride] =
                    padded[outer * padded_block + inner + (size_t)start * stride + (size_t)j * stride];
    return LSG_OK;
}

/* ---- upwind derivatives (spatial_derivatives.cpp:10-224) ---------------- */

int orc_ghost_width(int scheme) { /* :10-18 */
    switch (scheme) {
        case LSG_SCHEME_FIRST: return 1;
        case LSG_SCHEME_ENO2: return 2;
        case LSG_SCHEME_ENO3: return 3;
        case LSG_SCHEME_WENO5: return 3;
    }
    return -1;
}

int orc_min_nodes(int scheme) { /* :20-28 */
    switch (scheme) {
        case LSG_SCHEME_FIRST: return 3;
        case LSG_SCHEME_ENO2: return 5;
        case LSG_SCHEME_ENO3: return 7;
        case LSG_SCHEME_WENO5: return 7;
    }
    return -1;
}

static double minmag(double a, double b) { return fabs(a) <= fabs(b) ? a : b; } /* :32 */

/* :78-97 */
static double weno5_onesided(double v1, double v2, double v3, double v4, double v5) {
    const double eps = 1e-6;
    const double phi1 = v1 / 3.0 - 7.0 * v2 / 6.0 + 11.0 * v3 / 6.0;
    const double phi2 = -v2 / 6.0 + 5.0 * v3 / 6.0 + v4 / 3.0;
    const double phi3 = v3 / 3.0 + 5.0 * v4 / 6.0 - v5 / 6.0;
    const double s1 = (13.0 / 12.0) * (v1 - 2.0 * v2 + v3) * (v1 - 2.0 * v2 + v3) +
                      0.25 * (v1 - 4.0 * v2 + 3.0 * v3) * (v1 - 4.0 * v2 + 3.0 * v3);
    const double s2 = (13.0 / 12.0) * (v2 - 2.0 * v3 + v4) * (v2 - 2.0 * v3 + v4) + 0.25 * (v2 - v4) * (v2 - v4);
    const double s3 = (13.0 / 12.0) * (v3 - 2.0 * v4 + v5) * (v3 - 2.0 * v4 + v5) +
                      0.25 * (3.0 * v3 - 4.0 * v4 + v5) * (3.0 * v3 - 4.0 * v4 + v5);
    const double a1 = 0.1 / ((eps + s1) * (eps + s1));
    const double a2 = 0.6 / ((eps + s2) * (eps + s2));
    const double a3 = 0.3 / ((eps + s3) * (eps + s3));
    const double inv = 1.0 / (a1 + a2 + a3);
    return (a1 * phi1 + a2 * phi2 + a3 * phi3) * inv;
}

/* One padded line s (node i at s[i + width]) -> n left/right values. */
static void line_kernel(int scheme, const double* s, int n, double dx, double* d1, double* d2, double* d3,
                        double* left, double* right) {
    const double inv_dx = 1.0 / dx;
    if (scheme == LSG_SCHEME_FIRST) { /* :101-110 */
        for (int i = 0; i < n; ++i) {
            left[i] = (s[i + 1] - s[i]) * inv_dx;
            right[i] = (s[i + 2] - s[i + 1]) * inv_dx;
        }
    } else if (scheme == LSG_SCHEME_ENO2) { /* :112-134 */
        for (int k = 0; k <= n + 2; ++k) d1[k] = (s[k + 1] - s[k]) * inv_dx;
        for (int k = 1; k <= n + 2; ++k) d2[k] = (d1[k] - d1[k - 1]) * (0.5 * inv_dx);
        for (int i = 0; i < n; ++i) {
            const int si = i + 2;
            left[i] = d1[si - 1] + minmag(d2[si - 1], d2[si]) * dx;
            right[i] = d1[si] - minmag(d2[si], d2[si + 1]) * dx;
        }
    } else if (scheme == LSG_SCHEME_ENO3) { /* :136-197 */
        for (int k = 0; k <= n + 4; ++k) d1[k] = (s[k + 1] - s[k]) * inv_dx;
        for (int k = 1; k <= n + 4; ++k) d2[k] = (d1[k] - d1[k - 1]) * (0.5 * inv_dx);
        for (int k = 1; k <= n + 3; ++k) d3[k] = (d2[k + 1] - d2[k]) * (inv_dx / 3.0);
        const double dx2 = dx * dx;
        for (int i = 0; i < n; ++i) {
            const int si = i + 3;
            {
                const double q1 = d1[si - 1];
                int kstar;
                double c;
                if (fabs(d2[si - 1]) <= fabs(d2[si])) {
                    c = d2[si - 1];
                    kstar = si - 2;
                } else {
                    c = d2[si];
                    kstar = si - 1;
                }
                const double q2 = c * dx;
                const double cstar = minmag(d3[kstar], d3[kstar + 1]);
                const int istar = si - kstar;
                const double factor = (double)(3 * istar * istar - 6 * istar + 2);
                left[i] = q1 + q2 + cstar * factor * dx2;
            }
            {
                const double q1 = d1[si];
                int kstar;
                double c;
                if (fabs(d2[si]) <= fabs(d2[si + 1])) {
                    c = d2[si];
                    kstar = si - 1;
                } else {
                    c = d2[si + 1];
                    kstar = si;
                }
                const double q2 = -c * dx;
                const double cstar = minmag(d3[kstar], d3[kstar + 1]);
                const int istar = si - kstar;
                const double factor = (double)(3 * istar * istar - 6 * istar + 2);
                right[i] = q1 + q2 + cstar * factor * dx2;
            }
        }
    } else { /* WENO5 :199-214 */
        for (int k = 0; k <= n + 4; ++k) d1[k] = (s[k + 1] - s[k]) * inv_dx;
        for (int i = 0; i < n; ++i) {
            left[i] = weno5_onesided(d1[i], d1[i + 1], d1[i + 2], d1[i + 3], d1[i + 4]);
            right[i] = weno5_onesided(d1[i + 5], d1[i + 4], d1[i + 3], d1[i + 2], d1[i + 1]);
        }
    }
}

/* linewise (:37-74) + dispatch (:216-224) */
int orc_upwind(const lsg_grid* g, const double* v, int dim, int scheme, double* left, double* right) {
    int rc = orc_grid_check(g);
    if (rc) return rc;
    if (scheme < LSG_SCHEME_FIRST || scheme > LSG_SCHEME_WENO5) return fail(LSG_EINVAL, "unknown derivative scheme");
    if (dim < 0 || dim >= g->dim) return fail(LSG_EINVAL, "upwind: dimension out of range");
    const int n = g->counts[dim];
    if (n < orc_min_nodes(scheme))
        return fail(LSG_EINVAL, "upwind: needs at least %d nodes along dim %d", orc_min_nodes(scheme), dim);
    const int width = orc_ghost_width(scheme);
    const double dx = orc_spacing(g, dim);
    const size_t stride = stride_of(g, dim);
    const size_t line_block = stride * (size_t)n;
    const size_t n_outer = orc_node_count(g) / line_block;
    const size_t L = (size_t)(n + 2 * width + 8);
    double* buf = (double*)malloc(sizeof(double) * L * 6);
    double *s = buf, *d1 = buf + L, *d2 = buf + 2 * L, *d3 = buf + 3 * L, *ll = buf + 4 * L, *rl = buf + 5 * L;
    for (size_t outer = 0; outer < n_outer; ++outer)
        for (size_t inner = 0; inner < stride; ++inner) {
            const size_t base = outer * line_block + inner;
            orc_fill_padded_line(v, base, stride, n, width, bc_of(g, dim), s);
            line_kernel(scheme, s, n, dx, d1, d2, d3, ll, rl);
            for (int j = 0; j < n; ++j) {
                left[base + (size_t)j * stride] = ll[j];
                right[base + (size_t)j * stride] = rl[j];
            }
        }
    free(buf);
    return LSG_OK;
}

/* ---- Hamiltonians and dissipation bounds --------------------------------
 * Reference kinds: rockets reachability.cpp:12-66 (A.5), rotation :113-126.
 * Config kinds are builder-defined; same order as oracle/ref_driver.cpp. */

static double ham_value(const lsg_problem* p, int D, const double* x, const double* q) {
    const double* k = p->params;
    switch (p->kind) {
        case LSG_HAM_LINEAR: {
            double h = 0.0;
            for (int d = 0; d < D; ++d) h += k[d] * q[d];
            return h + k[12];
        }
        case LSG_HAM_ROTATION: return -x[1] * q[0] + x[0] * q[1];
        case LSG_HAM_ROCKETS: {
            const double a = k[0], gg = k[1], u_min = k[3], u_max = k[4];
            return -a * q[0] * cos(x[2]) - q[1] * (gg - a - a * sin(x[2])) - u_max * fabs(q[0] * x[0] + q[2]) +
                   u_min * fabs(q[1] * x[0] + q[2]);
        }
        case LSG_HAM_AIR3D: {
            const double va = k[0], vb = k[1], wa = k[2], wb = k[3];
            const double c = cos(x[2]), s = sin(x[2]);
            const double drift = ((-va) * q[0] + (vb * c) * q[0]) + (vb * s) * q[1];
            const double turn = wa * fabs((x[1] * q[0] - x[0] * q[1]) - q[2]);
            return -((drift + turn) - wb * fabs(q[2]));
        }
        case LSG_HAM_DBLINT4: return ((q[0] * x[1] + q[2] * x[3]) - fabs(q[1])) - fabs(q[3]);
        case LSG_HAM_DUBINS6: {
            const double ca = cos(x[2]), sa = sin(x[2]), cb = cos(x[5]), sb = sin(x[5]);
            return ((((q[0] * ca + q[1] * sa) + q[3] * cb) + q[4] * sb) - fabs(q[2])) + fabs(q[5]);
        }
        case LSG_HAM_NORMAL: {
            double r2 = 0.0;
            for (int d = 0; d < D; ++d) r2 += q[d] * q[d];
            return k[0] * sqrt(r2);
        }
    }
    return NAN;
}

static double bound_value(const lsg_problem* p, int dim, const double* x) {
    const double* k = p->params;
    switch (p->kind) {
        case LSG_HAM_LINEAR: return k[6 + dim];
        case LSG_HAM_ROTATION: return fabs(dim == 0 ? x[1] : x[0]);
        case LSG_HAM_ROCKETS: {
            const double a = k[0], gg = k[1], u_min = k[3], u_max = k[4];
            if (dim == 0) return fabs(a * cos(x[2])) + fabs(x[0]);
            if (dim == 1) return fabs(a * sin(x[2]) + a - gg) + fabs(x[0]);
            return u_max - u_min;
        }
        case LSG_HAM_AIR3D: {
            const double va = k[0], vb = k[1], wa = k[2], wb = k[3];
            if (dim == 0) return fabs(-va + vb * cos(x[2])) + wa * fabs(x[1]);
            if (dim == 1) return fabs(vb * sin(x[2])) + wa * fabs(x[0]);
            return wa + wb;
        }
        case LSG_HAM_DBLINT4: return dim == 0 ? fabs(x[1]) : dim == 2 ? fabs(x[3]) : 1.0;
        case LSG_HAM_DUBINS6: return 1.0;
        case LSG_HAM_NORMAL: return k[0];
    }
    return NAN;
}

static int check_problem(const lsg_grid* g, const lsg_problem* p) {
    if (!p) return fail(LSG_EINVAL, "term_lax_friedrichs: problem must provide ham_func and dissipation_bounds");
    if (p->scheme < LSG_SCHEME_FIRST || p->scheme > LSG_SCHEME_WENO5) return fail(LSG_EINVAL, "unknown derivative scheme");
    const int D = g->dim;
    switch (p->kind) {
        case LSG_HAM_LINEAR: case LSG_HAM_NORMAL: return LSG_OK;
        case LSG_HAM_ROTATION: return D == 2 ? LSG_OK : fail(LSG_EINVAL, "rotation: grid must be 2-D");
        case LSG_HAM_ROCKETS: return D == 3 ? LSG_OK : fail(LSG_EINVAL, "rocket_hamiltonian: grid must be 3-D (x, z, theta)");
        case LSG_HAM_AIR3D: return D == 3 ? LSG_OK : fail(LSG_EINVAL, "air3d: grid must be 3-D");
        case LSG_HAM_DBLINT4: return D == 4 ? LSG_OK : fail(LSG_EINVAL, "dblint4: grid must be 4-D");
        case LSG_HAM_DUBINS6: return D == 6 ? LSG_OK : fail(LSG_EINVAL, "dubins6: grid must be 6-D");
    }
    return fail(LSG_EINVAL, "term_lax_friedrichs: problem must provide ham_func and dissipation_bounds");
}

static void coords_of(const lsg_grid* g, double* const* axes, size_t i, double* x) {
    for (int d = 0; d < g->dim; ++d) {
        const size_t n = (size_t)g->counts[d];
        x[d] = axes[d][i % n];
        i /= n;
    }
}

/* ---- Lax-Friedrichs term (hamiltonian.cpp:11-88) ------------------------ */

int orc_term_lf(const lsg_grid* g, const lsg_problem* p, double t, const double* v, double* dvdt,
                double* step_bound) {
    (void)t;
    int rc = orc_grid_check(g);
    if (rc) return rc;
    if ((rc = check_problem(g, p))) return rc;
    const int D = g->dim;
    const size_t N = orc_node_count(g);
    double* L[LSG_MAX_DIM];
    double* R[LSG_MAX_DIM];
    double* axes[LSG_MAX_DIM];
    double* ham = (double*)malloc(sizeof(double) * N);
    for (int d = 0; d < D; ++d) {
        L[d] = (double*)malloc(sizeof(double) * N);
        R[d] = (double*)malloc(sizeof(double) * N);
        axes[d] = (double*)malloc(sizeof(double) * (size_t)g->counts[d]);
        orc_axis(g, d, axes[d]);
    }
    rc = LSG_OK;
    for (int d = 0; d < D && rc == LSG_OK; ++d) rc = orc_upwind(g, v, d, p->scheme, L[d], R[d]); /* :23-28 */
    double alpha[LSG_MAX_DIM] = {0};
    if (rc == LSG_OK) {
        double x[LSG_MAX_DIM], q[LSG_MAX_DIM];
        for (size_t i = 0; i < N; ++i) { /* central costate :31-32, H :36-40 */
            coords_of(g, axes, i, x);
            for (int d = 0; d < D; ++d) q[d] = 0.5 * (L[d][i] + R[d][i]);
            ham[i] = ham_value(p, D, x, q);
            if (!isfinite(ham[i])) {
                rc = fail(LSG_ENUMERIC, "term_lax_friedrichs: hamiltonian produced a non-finite value");
                break;
            }
        }
        for (int d = 0; d < D && rc == LSG_OK; ++d) { /* global LF alpha :44-56 */
            double m = 0.0;
            for (size_t i = 0; i < N; ++i) {
                coords_of(g, axes, i, x);
                const double b = bound_value(p, d, x);
                if (!isfinite(b) || b < 0.0) {
                    rc = fail(LSG_ENUMERIC, "term_lax_friedrichs: dissipation bound must be finite and non-negative");
                    break;
                }
                m = smax(m, b);
            }
            alpha[d] = m;
        }
    }
    if (rc == LSG_OK) {
        for (size_t i = 0; i < N; ++i) { /* combine :58-66 */
            double diss = 0.0;
            for (int d = 0; d < D; ++d) diss += alpha[d] * (R[d][i] - L[d][i]);
            double r = -(ham[i] - 0.5 * diss);
            if (p->restrict_update) /* :73-74, :78-88 */
                r = p->direction == LSG_GROW ? smin(r, 0.0) : smax(r, 0.0);
            dvdt[i] = r;
        }
        double speed = 0.0; /* :68-71 */
        for (int d = 0; d < D; ++d) speed += alpha[d] / orc_spacing(g, d);
        *step_bound = speed > 0.0 ? 1.0 / speed : INFINITY;
    }
    for (int d = 0; d < D; ++d) {
        free(L[d]);
        free(R[d]);
        free(axes[d]);
    }
    free(ham);
    return rc;
}

int orc_restrict_update(size_t n, const double* dvdt, int direction, double* out) {
    for (size_t i = 0; i < n; ++i) out[i] = direction == LSG_GROW ? smin(dvdt[i], 0.0) : smax(dvdt[i], 0.0);
    return LSG_OK;
}

/* ---- integrators (integrator.cpp:11-125) -------------------------------- */

static int check_options(const lsg_opts* o) { /* :11-20 */
    if (!(o->cfl_factor > 0.0)) return fail(LSG_EINVAL, "integrator: cfl_factor must be positive");
    if (!(o->max_step > 0.0)) return fail(LSG_EINVAL, "integrator: max_step must be positive");
    if (!(o->termination_epsilon > 0.0)) return fail(LSG_EINVAL, "integrator: termination_epsilon must be positive");
    for (size_t k = 1; k < o->n_checkpoint_times; ++k)
        if (o->checkpoint_times[k] < o->checkpoint_times[k - 1])
            return fail(LSG_EINVAL, "integrator: checkpoint_times must be ascending");
    return LSG_OK;
}

static const lsg_opts* opts_or_default(const lsg_opts* o, lsg_opts* tmp) {
    if (o) return o;
    tmp->cfl_factor = 0.32;
    tmp->max_step = INFINITY;
    tmp->termination_epsilon = 1e-6;
    tmp->checkpoint_times = NULL;
    tmp->n_checkpoint_times = 0;
    return tmp;
}

/* run_cfl :22-97 */
int orc_integrate(const lsg_grid* g, const lsg_problem* p, int method, double t0, double tf, double* v,
                  const lsg_opts* opts_in, lsg_steplog* steps, size_t cap, size_t* n_steps, double* t_final) {
    lsg_opts tmp;
    const lsg_opts* o = opts_or_default(opts_in, &tmp);
    int rc = orc_grid_check(g);
    if (rc) return rc;
    if (method < LSG_CFL1 || method > LSG_CFL3) return fail(LSG_EINVAL, "unknown integrator");
    if ((rc = check_options(o))) return rc;
    if (!isfinite(t0) || !isfinite(tf)) return fail(LSG_EINVAL, "integrator: tspan must be finite");
    if (tf < t0) return fail(LSG_EINVAL, "integrator: tspan must not be decreasing");
    size_t count = 0;
    double t = t0;
    if (tf != t0) {
        const size_t N = orc_node_count(g);
        const int order = method + 1;
        double* d1 = (double*)malloc(sizeof(double) * N);
        double* d2 = (double*)malloc(sizeof(double) * N);
        double* v1 = (double*)malloc(sizeof(double) * N);
        const double eps_stop = o->termination_epsilon * fabs(tf);
        while (tf - t > 0.0 && tf - t >= eps_stop) {
            double target = tf; /* :43-49 upper_bound */
            for (size_t k = 0; k < o->n_checkpoint_times; ++k)
                if (o->checkpoint_times[k] > t) {
                    if (o->checkpoint_times[k] < tf) target = o->checkpoint_times[k];
                    break;
                }
            double bound;
            if ((rc = orc_term_lf(g, p, t, v, d1, &bound))) break;
            const double remaining = target - t;
            double dt = smin(remaining, o->max_step);
            dt = smin(dt, o->cfl_factor * bound);
            if (!(dt > 0.0)) {
                rc = fail(LSG_ENUMERIC, "integrator: step size collapsed to zero");
                break;
            }
            const int lands = dt == remaining;
            if (order == 1) {
                for (size_t i = 0; i < N; ++i) v[i] += dt * d1[i];
            } else if (order == 2) {
                for (size_t i = 0; i < N; ++i) v1[i] = v[i] + dt * d1[i];
                double b2;
                if ((rc = orc_term_lf(g, p, t + dt, v1, d2, &b2))) break;
                for (size_t i = 0; i < N; ++i) v[i] += 0.5 * ((v1[i] + dt * d2[i]) - v[i]);
            } else {
                for (size_t i = 0; i < N; ++i) v1[i] = v[i] + dt * d1[i];
                double b2;
                if ((rc = orc_term_lf(g, p, t + dt, v1, d2, &b2))) break;
                for (size_t i = 0; i < N; ++i) v1[i] += dt * d2[i];
                for (size_t i = 0; i < N; ++i) v1[i] = v[i] + 0.25 * (v1[i] - v[i]); /* vhalf */
                if ((rc = orc_term_lf(g, p, t + 0.5 * dt, v1, d2, &b2))) break;
                for (size_t i = 0; i < N; ++i) {
                    const double v32 = v1[i] + dt * d2[i];
                    v[i] += (2.0 / 3.0) * (v32 - v[i]);
                }
            }
            double v_min = v[0], v_max = v[0];
            for (size_t i = 1; i < N; ++i) {
                v_min = smin(v_min, v[i]);
                v_max = smax(v_max, v[i]);
            }
            if (steps && count < cap) {
                lsg_steplog e = {t, dt, bound, v_min, v_max};
                steps[count] = e;
            }
            ++count;
            t = lands ? target : t + dt;
        }
        free(d1);
        free(d2);
        free(v1);
    }
    if (n_steps) *n_steps = count;
    if (t_final) *t_final = t;
    return rc;
}

/* solve_brt (reachability.cpp:135-174) */
int orc_solve_brt(const lsg_grid* g, const lsg_problem* p, const double* v0, double t_first, double t_second,
                  int n_checkpoints, int method, const lsg_opts* o, double* checkpoints, double* checkpoint_times,
                  int* n_out, lsg_steplog* steps, size_t cap, size_t* n_steps) {
    int rc = orc_grid_check(g);
    if (rc) return rc;
    if (n_checkpoints < 1) return fail(LSG_EINVAL, "solve_brt: need at least one checkpoint");
    if (!isfinite(t_first) || !isfinite(t_second)) return fail(LSG_EINVAL, "solve_brt: tspan must be finite");
    const size_t N = orc_node_count(g);
    const double duration = fabs(t_second - t_first);
    memcpy(checkpoints, v0, N * sizeof(double));
    checkpoint_times[0] = 0.0;
    *n_out = 1;
    size_t total = 0;
    if (!(duration == 0.0 || n_checkpoints == 1)) {
        const int segments = n_checkpoints - 1;
        double* v = (double*)malloc(N * sizeof(double));
        memcpy(v, v0, N * sizeof(double));
        double t = 0.0;
        for (int k = 1; k <= segments; ++k) {
            const double t_end = duration * (double)k / (double)segments;
            size_t leg_steps = 0;
            double leg_t;
            rc = orc_integrate(g, p, method, t, t_end, v, o, steps ? steps + (total < cap ? total : cap) : NULL,
                               cap > total ? cap - total : 0, &leg_steps, &leg_t);
            if (rc) break;
            total += leg_steps;
            t = leg_t;
            memcpy(checkpoints + (size_t)k * N, v, N * sizeof(double));
            checkpoint_times[k] = t_end;
            *n_out = k + 1;
        }
        free(v);
    }
    if (n_steps) *n_steps = total;
    return rc;
}

/* ---- implicit surfaces (implicit_surfaces.cpp:20-71) -------------------- */

int orc_cylinder(const lsg_grid* g, unsigned ignored_mask, const double* center, double radius, double* out) {
    int rc = orc_grid_check(g);
    if (rc) return rc;
    const size_t N = orc_node_count(g);
    double* axes[LSG_MAX_DIM];
    for (int d = 0; d < g->dim; ++d) {
        axes[d] = (double*)malloc(sizeof(double) * (size_t)g->counts[d]);
        orc_axis(g, d, axes[d]);
    }
    double x[LSG_MAX_DIM];
    for (size_t i = 0; i < N; ++i) {
        coords_of(g, axes, i, x);
        double r2 = 0.0;
        for (int d = 0; d < g->dim; ++d) {
            if (ignored_mask & (1u << d)) continue;
            const double dx = x[d] - center[d];
            r2 += dx * dx;
        }
        out[i] = sqrt(r2) - radius;
    }
    for (int d = 0; d < g->dim; ++d) free(axes[d]);
    return LSG_OK;
}

int orc_sphere(const lsg_grid* g, const double* center, double radius, double* out) {
    return orc_cylinder(g, 0u, center, radius, out);
}

/* implicit_surfaces.cpp:73-94 */
int orc_rectangle(const lsg_grid* g, const double* lower, const double* upper, double* out) {
    int rc = orc_grid_check(g);
    if (rc) return rc;
    for (int d = 0; d < g->dim; ++d)
        if (!(upper[d] > lower[d])) return fail(LSG_EINVAL, "rectangle: upper must exceed lower");
    const size_t N = orc_node_count(g);
    double* axes[LSG_MAX_DIM];
    for (int d = 0; d < g->dim; ++d) {
        axes[d] = (double*)malloc(sizeof(double) * (size_t)g->counts[d]);
        orc_axis(g, d, axes[d]);
    }
    double x[LSG_MAX_DIM];
    for (size_t i = 0; i < N; ++i) {
        coords_of(g, axes, i, x);
        double v = -INFINITY;
        for (int d = 0; d < g->dim; ++d) v = smax(v, smax(lower[d] - x[d], x[d] - upper[d]));
        out[i] = v;
    }
    for (int d = 0; d < g->dim; ++d) free(axes[d]);
    return LSG_OK;
}

/* implicit_surfaces.cpp:96-116 */
int orc_ellipsoid(const lsg_grid* g, double radius, double* out) {
    int rc = orc_grid_check(g);
    if (rc) return rc;
    if (g->dim != 2 && g->dim != 3) return fail(LSG_EINVAL, "ellipsoid: only 2-D and 3-D grids are supported");
    if (!(radius > 0.0)) return fail(LSG_EINVAL, "ellipsoid: radius must be positive");
    const size_t N = orc_node_count(g);
    double* axes[LSG_MAX_DIM];
    for (int d = 0; d < g->dim; ++d) {
        axes[d] = (double*)malloc(sizeof(double) * (size_t)g->counts[d]);
        orc_axis(g, d, axes[d]);
    }
    double x[LSG_MAX_DIM];
    for (size_t i = 0; i < N; ++i) {
        coords_of(g, axes, i, x);
        double v = x[0] * x[0] + 4.0 * x[1] * x[1];
        if (g->dim == 3) v += 9.0 * x[2] * x[2];
        out[i] = v - radius;
    }
    for (int d = 0; d < g->dim; ++d) free(axes[d]);
    return LSG_OK;
}

/* implicit_surfaces.cpp:128-151: op 1 union (std::min), 2 intersection (std::max), 3 complement */
int orc_set_op(const lsg_grid* g, int op, const double* a, const double* b, double* out) {
    int rc = orc_grid_check(g);
    if (rc) return rc;
    const size_t N = orc_node_count(g);
    for (size_t i = 0; i < N; ++i)
        out[i] = op == 1 ? smin(a[i], b[i]) : (op == 2 ? smax(a[i], b[i]) : -a[i]);
    return LSG_OK;
}
