/*
 * kpme_oracle.c -- CPU oracle (TEST INFRASTRUCTURE ONLY; see kpme_oracle.h).
 *
 * Restates, in plain C and in the reference's floating-point evaluation
 * order, the functions on the SKP-PME reciprocal path of
 * /root/reference/proj/include/kpme/. Each function cites the file:line it
 * follows. Build with -ffp-contract=off (oracle/Makefile).
 *
 * Storage differs from the reference in one place only: the per-rank factor
 * pairs of kpme_apply (parallel.hpp:261-279) are stored once per
 * (term, axis, cell index along that axis) instead of once per rank. build_uv
 * depends on nothing else, so the stored values are identical; this keeps
 * config 3/4 within host memory.
 */
#define _GNU_SOURCE
#include "kpme_oracle.h"

#include <complex.h>
#include <math.h>
#include <pthread.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

static __thread char g_err[512];

const char* ko_last_error(void) { return g_err; }

static int fail(int code, const char* msg) {
    snprintf(g_err, sizeof g_err, "%s", msg);
    return code;
}

/* ===================================================================== */
/* geometry.hpp                                                          */
/* ===================================================================== */

/* SeededUniform::next01, geometry.hpp:223-229 (splitmix64) */
static double next01(uint64_t* state) {
    uint64_t z = (*state += 0x9e3779b97f4a7c15ULL);
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    z ^= z >> 31;
    return (double)(z >> 11) * 0x1.0p-53;
}

/* sample_cloud, geometry.hpp:238-251 */
void ko_sample_cloud(const double center[3], double radius, int64_t n,
                     uint64_t seed, double* pos, double* q) {
    uint64_t s = seed;
    for (int64_t i = 0; i < n; ++i) {
        for (int a = 0; a < 3; ++a)
            pos[3 * i + a] = center[a] + radius * (2.0 * next01(&s) - 1.0);
        q[i] = 2.0 * next01(&s) - 1.0;
    }
}

/* CellGrid::axis_lo / axis_hi, geometry.hpp:90-98 */
static double axis_lo(const double* center, double radius, const int* counts,
                      int axis, int idx) {
    return center[axis] - radius + 2.0 * radius * idx / counts[axis];
}
static double axis_hi(const double* center, double radius, const int* counts,
                      int axis, int idx) {
    return center[axis] - radius + 2.0 * radius * (idx + 1) / counts[axis];
}

/* CellGrid::axis_nodes, geometry.hpp:102-110 */
static void axis_nodes(const double* center, double radius, const int* counts,
                       int axis, int idx, int order, double* nodes) {
    const double a = axis_lo(center, radius, counts, axis, idx);
    const double b = axis_hi(center, radius, counts, axis, idx);
    for (int k = 0; k < order; ++k) nodes[k] = a + (b - a) * k / (order - 1);
}

/* assign_particles, geometry.hpp:131-154 */
int ko_assign_particles(const double center[3], double radius,
                        const int counts[3], int64_t n, const double* pos,
                        int32_t* cell_of, int32_t* perm, int32_t* cell_start,
                        int64_t* bad_index) {
    const int ncell = counts[0] * counts[1] * counts[2];
    for (int c = 0; c <= ncell; ++c) cell_start[c] = 0;
    for (int64_t i = 0; i < n; ++i) {
        const double* p = pos + 3 * i;
        /* Box3::contains, geometry.hpp:36-40 */
        for (int a = 0; a < 3; ++a)
            if (fabs(p[a] - center[a]) > radius) {
                if (bad_index) *bad_index = i;
                snprintf(g_err, sizeof g_err,
                         "assign_particles: particle %lld outside the box",
                         (long long)i);
                return KO_INVALID_ARGUMENT;
            }
        int c[3];
        for (int a = 0; a < 3; ++a) {
            const int K = counts[a];
            const double t = (p[a] - (center[a] - radius)) * K / (2.0 * radius);
            int idx = (int)floor(t);
            if (t == (double)idx && idx > 0) --idx;
            if (idx < 0) idx = 0;
            if (idx > K - 1) idx = K - 1;
            c[a] = idx;
        }
        const int flat = (c[0] * counts[1] + c[1]) * counts[2] + c[2];
        cell_of[i] = flat;
        cell_start[flat + 1]++;
    }
    for (int c = 0; c < ncell; ++c) cell_start[c + 1] += cell_start[c];
    /* members are appended in ascending particle order */
    int32_t* cursor = (int32_t*)malloc(sizeof(int32_t) * (ncell + 1));
    memcpy(cursor, cell_start, sizeof(int32_t) * ncell);
    for (int64_t i = 0; i < n; ++i) perm[cursor[cell_of[i]]++] = (int32_t)i;
    free(cursor);
    return KO_OK;
}

/* ===================================================================== */
/* alpha.hpp                                                             */
/* ===================================================================== */

/* alpha_weight, alpha.hpp:34-39 */
double ko_alpha_weight(double xi, int m0, int m1, int m2) {
    const double r2 = (double)m0 * m0 + (double)m1 * m1 + (double)m2 * m2;
    if (r2 == 0.0) return 0.0;
    const double p = M_PI / xi;
    return exp(-p * p * r2) / r2;
}

/* quadrature_max_error, alpha.hpp:99-108 */
double ko_quadrature_max_error(int count, const double* nodes,
                               const double* weights, int64_t max_arg) {
    double worst = 0.0;
    for (int64_t r = 1; r <= max_arg; ++r) {
        double s = 0.0;
        for (int l = 0; l < count; ++l) s += weights[l] * exp(-nodes[l] * (double)r);
        const double e = fabs(1.0 / (double)r - s);
        worst = (worst < e) ? e : worst; /* std::max */
    }
    return worst;
}

/* sinc_rule, alpha.hpp:114-151 */
int ko_sinc_rule(int n_quad, int modes, double* nodes, double* weights,
                 double* lifting, double* eps) {
    if (n_quad < 1) return fail(KO_INVALID_ARGUMENT, "sinc_rule: n_quad must be >= 1");
    if (modes < 1) return fail(KO_INVALID_ARGUMENT, "sinc_rule: modes must be >= 1");
    const double h_star = M_PI / sqrt(2.0 * n_quad + 1.0);
    const int64_t max_arg = 3LL * modes * modes;
    const int count = 2 * n_quad + 1;
    double* tn = (double*)malloc(sizeof(double) * count);
    double* tw = (double*)malloc(sizeof(double) * count);
    double best_err = INFINITY, best_h = 0.0;
    int have = 0;
    const int candidates = 64;
    for (int c = 0; c < candidates; ++c) {
        const double t = (double)c / (candidates - 1);
        const double h = (h_star / 4.0) * pow(16.0, t);
        for (int l = -n_quad; l <= n_quad; ++l) {
            tw[l + n_quad] = h / (1.0 + exp(-l * h));
            tn[l + n_quad] = log1p(exp(l * h));
        }
        const double err = ko_quadrature_max_error(count, tn, tw, max_arg);
        if (err < best_err) {
            best_err = err;
            best_h = h;
            memcpy(nodes, tn, sizeof(double) * count);
            memcpy(weights, tw, sizeof(double) * count);
            have = 1;
        }
    }
    free(tn);
    free(tw);
    if (!have) { /* every candidate was NaN: the reference returns an empty rule */
        return fail(KO_NUMERICAL, "sinc_rule: no finite candidate");
    }
    if (lifting) *lifting = best_h;
    if (eps) *eps = best_err;
    return KO_OK;
}

/* sinc_rule_for_eps, alpha.hpp:154-161 */
int ko_sinc_rule_for_eps(double eps, int modes, int max_n, int* n_quad,
                         double* nodes, double* weights, double* lifting,
                         double* eps_out) {
    if (!(eps > 0.0))
        return fail(KO_INVALID_ARGUMENT, "sinc_rule_for_eps: eps must be positive");
    for (int n = 1; n <= max_n; ++n) {
        double h, e;
        const int st = ko_sinc_rule(n, modes, nodes, weights, &h, &e);
        if (st != KO_OK) return st;
        if (e <= eps) {
            *n_quad = n;
            if (lifting) *lifting = h;
            if (eps_out) *eps_out = e;
            return KO_OK;
        }
    }
    return fail(KO_NUMERICAL, "sinc_rule_for_eps: eps not reached within node budget");
}

/* skp_from_quadrature, alpha.hpp:165-188 */
int ko_skp_from_quadrature(int count, const double* nodes,
                           const double* weights, double min_arg,
                           double max_arg, double xi, int modes,
                           double* term_weights, double* profiles,
                           double* correction) {
    const int M = modes;
    if (!(min_arg <= 1.0 && max_arg >= 3.0 * M * M))
        return fail(KO_INVALID_ARGUMENT,
                    "skp_from_quadrature: rule does not cover arguments [1, 3M^2]");
    const double shift = (M_PI / xi) * (M_PI / xi);
    const int P = 2 * M + 1;
    double corr = 0.0;
    for (int l = 0; l < count; ++l) {
        term_weights[l] = weights[l];
        for (int m = -M; m <= M; ++m) {
            const double v = exp(-(nodes[l] + shift) * (double)m * (double)m);
            for (int a = 0; a < 3; ++a) profiles[((int64_t)l * 3 + a) * P + m + M] = v;
        }
        corr += weights[l];
    }
    *correction = corr;
    return KO_OK;
}

/* optimal_term_lower_bound, alpha.hpp:286-291 */
int64_t ko_optimal_term_lower_bound(double eps) {
    if (!(eps > 0.0 && eps < 16.0)) {
        fail(KO_INVALID_ARGUMENT, "optimal_term_lower_bound: need 0 < eps < 16");
        return -1;
    }
    const double t = log(eps / 16.0) / M_PI;
    return (int64_t)ceil(t * t - 1e-9);
}

/* ===================================================================== */
/* interpolation.hpp                                                     */
/* ===================================================================== */

/* lagrange_weights_1d, interpolation.hpp:20-36 */
int ko_lagrange_weights_1d(int order, double a, double b, double y, double* w) {
    if (order < 2) return fail(KO_INVALID_ARGUMENT, "lagrange_weights_1d: order must be >= 2");
    if (a == b) return fail(KO_INVALID_ARGUMENT, "lagrange_weights_1d: degenerate interval");
    const double t = (y - 0.5 * (b + a)) / (0.5 * (b - a));
    for (int k = 0; k < order; ++k) {
        const double tk = -1.0 + 2.0 * k / (order - 1);
        double prod = 1.0;
        for (int j = 0; j < order; ++j) {
            if (j == k) continue;
            const double tj = -1.0 + 2.0 * j / (order - 1);
            prod *= (t - tj) / (tk - tj);
        }
        w[k] = prod;
    }
    return KO_OK;
}

/* tensor_weights, interpolation.hpp:40-59; w has order^3 entries */
static int tensor_weights(const double* center, double radius, const int* counts,
                          const int cell[3], int order, const double* y,
                          double* w) {
    double w1[3][64];
    for (int a = 0; a < 3; ++a) {
        const double lo = axis_lo(center, radius, counts, a, cell[a]);
        const double hi = axis_hi(center, radius, counts, a, cell[a]);
        const double slack = 1e-12 * (hi - lo);
        if (y[a] < lo - slack || y[a] > hi + slack)
            return fail(KO_INVALID_ARGUMENT, "tensor_weights: point outside cell");
        const int st = ko_lagrange_weights_1d(order, lo, hi, y[a], w1[a]);
        if (st) return st;
    }
    int64_t idx = 0;
    for (int i = 0; i < order; ++i)
        for (int j = 0; j < order; ++j)
            for (int k = 0; k < order; ++k) w[idx++] = w1[0][i] * w1[1][j] * w1[2][k];
    return KO_OK;
}

/* ===================================================================== */
/* symfourier.hpp                                                        */
/* ===================================================================== */

/* build_w, symfourier.hpp:23-33 */
int ko_build_w(int m, int npts, const double* pts, double* w) {
    if (m < 0) return fail(KO_INVALID_ARGUMENT, "build_w: m must be >= 0");
    const double scale = m == 0 ? 1.0 : sqrt(2.0);
    for (int j = 0; j < npts; ++j) {
        const double ph = 2.0 * M_PI * m * pts[j];
        w[j] = scale * cos(ph);
        w[npts + j] = scale * sin(ph);
    }
    return KO_OK;
}

/* even_profile, symfourier.hpp:69-71 */
static double even_profile(const double* p, int m, int modes) {
    return 0.5 * (p[m + modes] + p[modes - m]);
}

/* build_uv, symfourier.hpp:108-124 (target nodes == source nodes) */
int ko_build_uv(double weight, const double* profile, int L,
                const double* nodes, int modes, double* u, double* v) {
    const int R = 2 * (modes + 1);
    const double ws = cbrt(weight);
    double w[2 * 64];
    for (int m = 0; m <= modes; ++m) {
        ko_build_w(m, L, nodes, w);
        const double s = ws * even_profile(profile, m, modes);
        for (int j = 0; j < L; ++j) {
            u[j * R + 2 * m] = w[j];
            u[j * R + 2 * m + 1] = w[L + j];
            v[(2 * m) * L + j] = s * w[j];
            v[(2 * m + 1) * L + j] = s * w[L + j];
        }
    }
    return KO_OK;
}

/* ===================================================================== */
/* kron.hpp                                                              */
/* ===================================================================== */

/* matricize, kron.hpp:39-58: m is rows x (total/rows) row-major */
static void matricize(const double* v, int d, const int* shape, int k, double* m) {
    int64_t total = 1, inner = 1;
    for (int a = 0; a < d; ++a) total *= shape[a];
    for (int a = k + 1; a < d; ++a) inner *= shape[a];
    const int64_t rows = shape[k], cols = total / rows, outer = total / (rows * inner);
    for (int64_t o = 0; o < outer; ++o)
        for (int64_t r = 0; r < rows; ++r)
            for (int64_t i = 0; i < inner; ++i)
                m[r * cols + o * inner + i] = v[(o * rows + r) * inner + i];
}

/* vectorize, kron.hpp:61-81 */
static void vectorize(const double* m, int d, const int* shape, int k, double* v) {
    int64_t total = 1, inner = 1;
    for (int a = 0; a < d; ++a) total *= shape[a];
    for (int a = k + 1; a < d; ++a) inner *= shape[a];
    const int64_t rows = shape[k], cols = total / rows, outer = total / (rows * inner);
    for (int64_t o = 0; o < outer; ++o)
        for (int64_t r = 0; r < rows; ++r)
            for (int64_t i = 0; i < inner; ++i)
                v[(o * rows + r) * inner + i] = m[r * cols + o * inner + i];
}

/* Dense product C = A * B, every entry summed over k ascending from 0.0
 * (the evaluation order of the Eigen subset oracle/_ref is built with). */
static void matmul(const double* A, const double* B, double* C, int64_t M,
                   int64_t K, int64_t N) {
    for (int64_t i = 0; i < M * N; ++i) C[i] = 0.0;
    for (int64_t i = 0; i < M; ++i)
        for (int64_t k = 0; k < K; ++k) {
            const double a = A[i * K + k];
            const double* b = B + k * N;
            double* c = C + i * N;
            for (int64_t j = 0; j < N; ++j) c[j] += a * b[j];
        }
}

/* kron_matvec_shuffle, kron.hpp:180-197 with dense KronFactor::apply
 * (kron.hpp:109-122) */
int ko_kron_matvec_shuffle(int d, const int* rows, const int* cols,
                           const double* const* factors, const double* q,
                           double* out, int64_t* multiplies) {
    if (d == 0) return fail(KO_INVALID_ARGUMENT, "kron_matvec_shuffle: empty operand");
    int shape[16];
    int64_t cap = 1, total = 1;
    for (int p = 0; p < d; ++p) {
        shape[p] = cols[p];
        total *= cols[p];
    }
    /* largest intermediate */
    {
        int s[16];
        memcpy(s, shape, sizeof(int) * d);
        int64_t t = total;
        cap = t;
        for (int p = d - 1; p >= 0; --p) {
            t = t / s[p] * rows[p];
            s[p] = rows[p];
            if (t > cap) cap = t;
        }
    }
    double* v = (double*)malloc(sizeof(double) * cap);
    double* m = (double*)malloc(sizeof(double) * cap);
    double* r = (double*)malloc(sizeof(double) * cap);
    memcpy(v, q, sizeof(double) * total);
    int64_t mult = 0;
    for (int p = d - 1; p >= 0; --p) {
        matricize(v, d, shape, p, m);
        const int64_t mc = total / shape[p];
        matmul(factors[p], m, r, rows[p], cols[p], mc);
        mult += (int64_t)rows[p] * cols[p] * mc;
        total = mc * rows[p];
        shape[p] = rows[p];
        vectorize(r, d, shape, p, v);
    }
    memcpy(out, v, sizeof(double) * total);
    free(v);
    free(m);
    free(r);
    if (multiplies) *multiplies = mult;
    return KO_OK;
}

/* op_count_estimate, kron.hpp:201-211 */
int64_t ko_op_count_estimate(int d, const int* rows, const int* cols) {
    int64_t total = 0;
    for (int p = 0; p < d; ++p) {
        int64_t c = 1;
        for (int k = 0; k < p; ++k) c *= cols[k];
        for (int k = p + 1; k < d; ++k) c *= rows[k];
        total += (int64_t)rows[p] * cols[p] * c;
    }
    return total;
}

/* ===================================================================== */
/* parallel.hpp                                                          */
/* ===================================================================== */

/* parallel_for, parallel.hpp:31-44: strided split over std::threads */
typedef void (*body_fn)(int i, void* ctx);
typedef struct { int t, nt, n; body_fn fn; void* ctx; } pf_slot;
static void* pf_run(void* arg) {
    pf_slot* s = (pf_slot*)arg;
    for (int i = s->t; i < s->n; i += s->nt) s->fn(i, s->ctx);
    return NULL;
}
static void parallel_for(int n, int threads, body_fn fn, void* ctx) {
    if (threads <= 1 || n <= 1) {
        for (int i = 0; i < n; ++i) fn(i, ctx);
        return;
    }
    const int nt = threads < n ? threads : n;
    pthread_t* th = (pthread_t*)malloc(sizeof(pthread_t) * nt);
    pf_slot* slots = (pf_slot*)malloc(sizeof(pf_slot) * nt);
    for (int t = 0; t < nt; ++t) {
        slots[t] = (pf_slot){t, nt, n, fn, ctx};
        pthread_create(&th[t], NULL, pf_run, &slots[t]);
    }
    for (int t = 0; t < nt; ++t) pthread_join(th[t], NULL);
    free(th);
    free(slots);
}

/* ledger (parallel.hpp:84-89) */
typedef struct {
    int64_t* rows;
    int64_t cap, count;
    int step;
} ledger_t;
static void ledger_push(ledger_t* l, int rank, int step, int axis, int64_t payload) {
    if (l->rows && l->count < l->cap) {
        int64_t* r = l->rows + 4 * l->count;
        r[0] = rank;
        r[1] = step;
        r[2] = axis;
        r[3] = payload;
    }
    l->count++;
}

/* Problem state shared by the stages of kpme_apply. */
typedef struct {
    const ko_apply_args* a;
    int K[3], ncell, L, L3, R, M, nt;
    int32_t* cell_of;
    int32_t* perm;
    int32_t* start;
    double* weights;  /* [n][L^3], InterpOperator::weights_ */
    double* U;        /* [3][K_a][L x R], lambda-free target factor */
    double* V;        /* [nterms][3][K_a][R x L] */
    int64_t uoff[3], voff[3];
} problem_t;

static void problem_free(problem_t* P) {
    free(P->cell_of);
    free(P->perm);
    free(P->start);
    free(P->weights);
    free(P->U);
    free(P->V);
}

static void unflatten(const int* K, int idx, int c[3]) {
    c[2] = idx % K[2];
    idx /= K[2];
    c[1] = idx % K[1];
    c[0] = idx / K[1];
}
static int flatten(const int* K, const int c[3]) { return (c[0] * K[1] + c[1]) * K[2] + c[2]; }

/* kpme_apply prologue: argument checks (parallel.hpp:247-248), partition
 * (geometry.hpp:131), InterpOperator ctor (interpolation.hpp:65-74) and the
 * factor loop (parallel.hpp:261-279, de-duplicated, see file header). */
static int problem_init(problem_t* P, const ko_apply_args* a, int need_particles) {
    memset(P, 0, sizeof *P);
    P->a = a;
    if (a->dec_modes != a->modes)
        return fail(KO_INVALID_ARGUMENT, "kpme_apply: decomposition mode bound mismatch");
    if (!(a->xi > 0.0)) return fail(KO_INVALID_ARGUMENT, "EwaldConfig: xi must be positive");
    if (a->modes < 1) return fail(KO_INVALID_ARGUMENT, "EwaldConfig: modes must be >= 1");
    if (!(a->radius > 0.0)) return fail(KO_INVALID_ARGUMENT, "Box3: radius must be positive");
    for (int d = 0; d < 3; ++d)
        if (a->counts[d] < 1)
            return fail(KO_INVALID_ARGUMENT, "build_cell_grid: cell counts must be >= 1");
    if (a->order < 2)
        return fail(KO_INVALID_ARGUMENT, "CellGrid: interpolation order must be >= 2");
    if (a->order > 64) return fail(KO_INVALID_ARGUMENT, "oracle: order > 64 unsupported");
    for (int d = 0; d < 3; ++d) P->K[d] = a->counts[d];
    P->ncell = P->K[0] * P->K[1] * P->K[2];
    P->L = a->order;
    P->L3 = P->L * P->L * P->L;
    P->M = a->modes;
    P->R = 2 * (P->M + 1);
    P->nt = a->nterms;
    const int L = P->L, R = P->R;

    if (need_particles) {
        P->cell_of = (int32_t*)malloc(sizeof(int32_t) * (a->n > 0 ? a->n : 1));
        P->perm = (int32_t*)malloc(sizeof(int32_t) * (a->n > 0 ? a->n : 1));
        P->start = (int32_t*)malloc(sizeof(int32_t) * (P->ncell + 1));
        int64_t bad = -1;
        int st = ko_assign_particles(a->center, a->radius, a->counts, a->n, a->pos,
                                     P->cell_of, P->perm, P->start, &bad);
        if (st) return st;
        P->weights = (double*)malloc(sizeof(double) * (a->n > 0 ? a->n : 1) * P->L3);
        for (int c = 0; c < P->ncell; ++c) {
            int mi[3];
            unflatten(P->K, c, mi);
            for (int32_t s = P->start[c]; s < P->start[c + 1]; ++s) {
                const int32_t p = P->perm[s];
                st = tensor_weights(a->center, a->radius, a->counts, mi, L,
                                    a->pos + 3 * (int64_t)p,
                                    P->weights + (int64_t)p * P->L3);
                if (st) return st;
            }
        }
    }

    /* factors: U[a][i] (L x R), V[t][a][i] (R x L) */
    int64_t usz = 0, vsz = 0;
    for (int d = 0; d < 3; ++d) {
        P->uoff[d] = usz;
        P->voff[d] = vsz;
        usz += (int64_t)P->K[d] * L * R;
        vsz += (int64_t)P->K[d] * R * L;
    }
    P->U = (double*)malloc(sizeof(double) * (usz > 0 ? usz : 1));
    P->V = (double*)malloc(sizeof(double) * (vsz * (P->nt > 0 ? P->nt : 1)));
    const int Pm = 2 * P->M + 1;
    double nodes[64];
    double* scratch_u = (double*)malloc(sizeof(double) * L * R);
    for (int d = 0; d < 3; ++d)
        for (int i = 0; i < P->K[d]; ++i) {
            axis_nodes(a->center, a->radius, a->counts, d, i, L, nodes);
            for (int k = 0; k < L; ++k) nodes[k] -= a->center[d];
            for (int t = 0; t < P->nt; ++t) {
                double* u = (t == 0) ? P->U + P->uoff[d] + (int64_t)i * L * R : scratch_u;
                double* v = P->V + (int64_t)t * vsz + P->voff[d] + (int64_t)i * R * L;
                ko_build_uv(a->term_weights[t], a->profiles + ((int64_t)t * 3 + d) * Pm, L,
                            nodes, P->M, u, v);
            }
            if (P->nt == 0) { /* U is lambda-free; build it even without terms */
                const int Rr = R;
                double w[2 * 64];
                for (int m = 0; m <= P->M; ++m) {
                    ko_build_w(m, L, nodes, w);
                    for (int j = 0; j < L; ++j) {
                        P->U[P->uoff[d] + (int64_t)i * L * Rr + j * Rr + 2 * m] = w[j];
                        P->U[P->uoff[d] + (int64_t)i * L * Rr + j * Rr + 2 * m + 1] = w[L + j];
                    }
                }
            }
        }
    free(scratch_u);
    return KO_OK;
}

static const double* Ufac(const problem_t* P, int axis, int i) {
    return P->U + P->uoff[axis] + (int64_t)i * P->L * P->R;
}
static const double* Vfac(const problem_t* P, int t, int axis, int i) {
    int64_t vsz = P->voff[2] + (int64_t)P->K[2] * P->R * P->L;
    return P->V + (int64_t)t * vsz + P->voff[axis] + (int64_t)i * P->R * P->L;
}

/* InterpOperator::interpolate, interpolation.hpp:84-92 */
static void do_interpolate(const problem_t* P, const double* q, double* phi) {
    memset(phi, 0, sizeof(double) * P->ncell * P->L3);
    for (int c = 0; c < P->ncell; ++c) {
        double* out = phi + (int64_t)c * P->L3;
        for (int32_t s = P->start[c]; s < P->start[c + 1]; ++s) {
            const int32_t p = P->perm[s];
            const double* w = P->weights + (int64_t)p * P->L3;
            const double qp = q[p];
            for (int i = 0; i < P->L3; ++i) out[i] = out[i] + qp * w[i];
        }
    }
}

/* InterpOperator::anterpolate, interpolation.hpp:95-105 */
static void do_anterpolate(const problem_t* P, const double* psi, double* out) {
    for (int c = 0; c < P->ncell; ++c) {
        const double* g = psi + (int64_t)c * P->L3;
        for (int32_t s = P->start[c]; s < P->start[c + 1]; ++s) {
            const int32_t p = P->perm[s];
            const double* w = P->weights + (int64_t)p * P->L3;
            double acc = 0.0;
            for (int i = 0; i < P->L3; ++i) acc += w[i] * g[i];
            out[p] = acc;
        }
    }
}

/* SimulatedComm::allreduce_axis, parallel.hpp:110-127: groups are the ranks
 * that agree on every other axis; sums run in ascending rank order. buf holds
 * ncell blocks of `len` doubles. */
static void allreduce_axis(const problem_t* P, ledger_t* led, int axis,
                           double* buf, int64_t len) {
    const int step = led->step++;
    const int Ka = P->K[axis];
    double* sum = (double*)malloc(sizeof(double) * len);
    char* done = (char*)calloc(P->ncell, 1);
    for (int r = 0; r < P->ncell; ++r) {
        if (done[r]) continue;
        int c[3];
        unflatten(P->K, r, c);
        c[axis] = 0;
        const int g0 = flatten(P->K, c);
        memcpy(sum, buf + (int64_t)g0 * len, sizeof(double) * len);
        for (int g = 1; g < Ka; ++g) {
            c[axis] = g;
            const double* src = buf + (int64_t)flatten(P->K, c) * len;
            for (int64_t i = 0; i < len; ++i) sum[i] += src[i];
        }
        for (int g = 0; g < Ka; ++g) {
            c[axis] = g;
            const int member = flatten(P->K, c);
            memcpy(buf + (int64_t)member * len, sum, sizeof(double) * len);
            done[member] = 1;
        }
    }
    free(sum);
    free(done);
    for (int r = 0; r < P->ncell; ++r) ledger_push(led, r, step, axis, len);
}

/* local V / U phases of spkmv (parallel.hpp:169-176), run by parallel_for */
typedef struct {
    const problem_t* P;
    int p, t0, nt_block;   /* axis, first term, number of stacked terms */
    double* const* data;   /* data[t] -> [ncell][L^3] */
    double* buf;           /* [ncell][nt_block*R][L^2] */
} phase_ctx;

static void v_phase(int r, void* vctx) {
    phase_ctx* x = (phase_ctx*)vctx;
    const problem_t* P = x->P;
    const int L = P->L, L2 = L * L, R = P->R;
    const int shape[3] = {L, L, L};
    int c[3];
    unflatten(P->K, r, c);
    double* m = (double*)malloc(sizeof(double) * P->L3);
    for (int tb = 0; tb < x->nt_block; ++tb) {
        matricize(x->data[tb] + (int64_t)r * P->L3, 3, shape, x->p, m);
        matmul(Vfac(P, x->t0 + tb, x->p, c[x->p]), m,
               x->buf + ((int64_t)r * x->nt_block + tb) * R * L2, R, L, L2);
    }
    free(m);
}

static void u_phase(int r, void* vctx) {
    phase_ctx* x = (phase_ctx*)vctx;
    const problem_t* P = x->P;
    const int L = P->L, L2 = L * L, R = P->R;
    const int shape[3] = {L, L, L};
    int c[3];
    unflatten(P->K, r, c);
    double* res = (double*)malloc(sizeof(double) * P->L3);
    for (int tb = 0; tb < x->nt_block; ++tb) {
        matmul(Ufac(P, x->p, c[x->p]), x->buf + ((int64_t)r * x->nt_block + tb) * R * L2,
               res, L, R, L2);
        vectorize(res, 3, shape, x->p, x->data[tb] + (int64_t)r * P->L3);
    }
    free(res);
}

/* spkmv (parallel.hpp:156-179) for terms [t0, t0+nt_block) stacked; with
 * nt_block == 1 this is one per-term spkmv, with nt_block == |Lambda| it is
 * the fused branch of spkmv_sum (parallel.hpp:200-227). */
static void spkmv_block(const problem_t* P, ledger_t* led, int t0, int nt_block,
                        double* const* data) {
    const int L2 = P->L * P->L;
    const int64_t len = (int64_t)nt_block * P->R * L2;
    double* buf = (double*)malloc(sizeof(double) * P->ncell * len);
    for (int p = 2; p >= 0; --p) {
        phase_ctx x = {P, p, t0, nt_block, data, buf};
        parallel_for(P->ncell, P->a->threads, v_phase, &x);
        allreduce_axis(P, led, p, buf, len);
        parallel_for(P->ncell, P->a->threads, u_phase, &x);
    }
    free(buf);
}

/* spkmv_sum, parallel.hpp:184-228 */
static void do_spkmv_sum(const problem_t* P, ledger_t* led, const double* phi,
                         double* psi) {
    const int64_t sz = (int64_t)P->ncell * P->L3;
    memset(psi, 0, sizeof(double) * sz);
    if (P->nt == 0) return;
    if (!P->a->fuse_terms) {
        double* z = (double*)malloc(sizeof(double) * sz);
        for (int t = 0; t < P->nt; ++t) {
            memcpy(z, phi, sizeof(double) * sz);
            double* d[1] = {z};
            spkmv_block(P, led, t, 1, d);
            for (int64_t i = 0; i < sz; ++i) psi[i] += z[i];
        }
        free(z);
        return;
    }
    double** d = (double**)malloc(sizeof(double*) * P->nt);
    for (int t = 0; t < P->nt; ++t) {
        d[t] = (double*)malloc(sizeof(double) * sz);
        memcpy(d[t], phi, sizeof(double) * sz);
    }
    spkmv_block(P, led, 0, P->nt, d);
    /* out[r] += data[t][r], terms ascending */
    for (int t = 0; t < P->nt; ++t) {
        for (int64_t i = 0; i < sz; ++i) psi[i] += d[t][i];
        free(d[t]);
    }
    free(d);
}

/* kpme_apply, parallel.hpp:243-290 */
int ko_kpme_apply(const ko_apply_args* a, double* potentials, int64_t* ledger,
                  int64_t ledger_cap, int64_t* ledger_rows) {
    problem_t P;
    int st = problem_init(&P, a, 1);
    if (st) {
        problem_free(&P);
        return st;
    }
    ledger_t led = {ledger, ledger_cap, 0, 0};

    /* local charges + allreduce_scalar (parallel.hpp:254-257, 130-138) */
    double total = 0.0;
    {
        const int step = led.step++;
        for (int r = 0; r < P.ncell; ++r) {
            double lc = 0.0;
            for (int32_t s = P.start[r]; s < P.start[r + 1]; ++s) lc += a->q[P.perm[s]];
            total += lc;
        }
        for (int r = 0; r < P.ncell; ++r) ledger_push(&led, r, step, -1, 1);
    }

    const int64_t sz = (int64_t)P.ncell * P.L3;
    double* phi = (double*)malloc(sizeof(double) * sz);
    double* psi = (double*)malloc(sizeof(double) * sz);
    do_interpolate(&P, a->q, phi);
    do_spkmv_sum(&P, &led, phi, psi);
    do_anterpolate(&P, psi, potentials);
    const double correction = a->correction * total;
    for (int64_t i = 0; i < a->n; ++i) potentials[i] -= correction;
    if (ledger_rows) *ledger_rows = led.count;
    free(phi);
    free(psi);
    problem_free(&P);
    return KO_OK;
}

int ko_interpolate(const ko_apply_args* a, double* phi_cells) {
    problem_t P;
    int st = problem_init(&P, a, 1);
    if (!st) do_interpolate(&P, a->q, phi_cells);
    problem_free(&P);
    return st;
}

int ko_spkmv_sum(const ko_apply_args* a, const double* phi_cells, double* psi_cells) {
    problem_t P;
    int st = problem_init(&P, a, 0);
    if (!st) {
        ledger_t led = {NULL, 0, 0, 0};
        do_spkmv_sum(&P, &led, phi_cells, psi_cells);
    }
    problem_free(&P);
    return st;
}

int ko_anterpolate(const ko_apply_args* a, const double* psi_cells, double* out) {
    problem_t P;
    int st = problem_init(&P, a, 1);
    if (!st) do_anterpolate(&P, psi_cells, out);
    problem_free(&P);
    return st;
}

/* ===================================================================== */
/* oracle.hpp                                                            */
/* ===================================================================== */

/* dense_reciprocal_apply, oracle.hpp:21-58 */
int ko_dense_reciprocal_apply(int64_t n, const double* pos, const double* q,
                              double xi, int modes, double* out) {
    const int M = modes;
    const double nmodes = pow(2.0 * M + 1.0, 3);
    if ((double)n * (double)n * nmodes > 1e9)
        return fail(KO_INVALID_ARGUMENT, "dense_reciprocal_apply: size guard exceeded");
    for (int64_t i = 0; i < n; ++i) {
        double acc_re = 0.0, acc_im = 0.0, scale = 0.0;
        const double* x = pos + 3 * i;
        for (int64_t j = 0; j < n; ++j) {
            const double* y = pos + 3 * j;
            for (int m0 = -M; m0 <= M; ++m0)
                for (int m1 = -M; m1 <= M; ++m1)
                    for (int m2 = -M; m2 <= M; ++m2) {
                        const double al = ko_alpha_weight(xi, m0, m1, m2);
                        if (al == 0.0) continue;
                        const double ph = 2.0 * M_PI *
                                          (m0 * (x[0] - y[0]) + m1 * (x[1] - y[1]) +
                                           m2 * (x[2] - y[2]));
                        const double s = q[j] * al;
                        const double re = s * cos(ph), im = s * sin(ph);
                        acc_re += re;
                        acc_im += im;
                        scale += hypot(re, im);
                    }
        }
        if (fabs(acc_im) > 1e-12 * (scale > 1.0 ? scale : 1.0))
            return fail(KO_NUMERICAL, "dense_reciprocal_apply: imaginary residue too large");
        out[i] = acc_re;
    }
    return KO_OK;
}
