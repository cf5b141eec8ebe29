/*
 * kpme_oracle.h -- CPU oracle for the SKP-PME reciprocal hot path.
 *
 * TEST INFRASTRUCTURE ONLY. This is a plain-C restatement of the reference
 * algorithm (/root/reference/proj/include/kpme/ headers) used as the parity
 * checker by tests/, by __graft_entry__.smoke() and by bench.py's
 * cpu_baseline leg. The product path (paper_2601_18838_b200/, include/) never
 * links, imports or calls anything in this directory.
 *
 * Parity pin: tests/test_oracle_pins.py checks this oracle bit-for-bit
 * against the reference's own headers compiled here (oracle/_ref, built by
 * oracle/ref/Makefile against a clean-room Eigen subset) and against the
 * golden vectors in tests/golden/ produced by tests/golden/gen_golden.py.
 *
 * All floating-point expressions keep the reference's evaluation order and
 * are compiled with -ffp-contract=off so no FMA contraction changes rounding.
 */
#ifndef KPME_ORACLE_H
#define KPME_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* status codes shared with the product C-ABI (include/kpme_gpu.h) */
enum { KO_OK = 0, KO_INVALID_ARGUMENT = 1, KO_RUNTIME = 2, KO_NUMERICAL = 3 };

const char* ko_last_error(void);

/* ---- geometry.hpp ---------------------------------------------------- */
/* sample_cloud (geometry.hpp:238-251): pos is n*3 AoS, q is n */
void ko_sample_cloud(const double center[3], double radius, int64_t n,
                     uint64_t seed, double* pos, double* q);
/* assign_particles (geometry.hpp:131-154). Outputs: cell_of[n] (flattened
 * cell), perm[n] = concatenation of Partition.members in flattened cell
 * order, cell_start[K0*K1*K2 + 1]. On a particle outside the box returns
 * KO_INVALID_ARGUMENT with *bad_index = that particle. */
int ko_assign_particles(const double center[3], double radius,
                        const int counts[3], int64_t n, const double* pos,
                        int32_t* cell_of, int32_t* perm, int32_t* cell_start,
                        int64_t* bad_index);

/* ---- alpha.hpp ------------------------------------------------------- */
double ko_alpha_weight(double xi, int m0, int m1, int m2);
double ko_quadrature_max_error(int count, const double* nodes,
                               const double* weights, int64_t max_arg);
/* sinc_rule (alpha.hpp:114-151): nodes/weights sized 2*n_quad+1 */
int ko_sinc_rule(int n_quad, int modes, double* nodes, double* weights,
                 double* lifting, double* eps);
/* sinc_rule_for_eps (alpha.hpp:154-161): writes *n_quad; nodes/weights must
 * hold 2*max_n+1 entries */
int ko_sinc_rule_for_eps(double eps, int modes, int max_n, int* n_quad,
                         double* nodes, double* weights, double* lifting,
                         double* eps_out);
/* skp_from_quadrature (alpha.hpp:165-188): term_weights[count],
 * profiles[count][3][2M+1]; min/max_arg describe rule coverage */
int ko_skp_from_quadrature(int count, const double* nodes,
                           const double* weights, double min_arg,
                           double max_arg, double xi, int modes,
                           double* term_weights, double* profiles,
                           double* correction);
int64_t ko_optimal_term_lower_bound(double eps);

/* ---- interpolation.hpp ----------------------------------------------- */
int ko_lagrange_weights_1d(int order, double a, double b, double y, double* w);

/* ---- symfourier.hpp -------------------------------------------------- */
/* build_w (symfourier.hpp:23-33): w is 2 x npts row-major */
int ko_build_w(int m, int npts, const double* pts, double* w);
/* build_uv (symfourier.hpp:108-124) for target == source nodes:
 * u is L x 2(M+1) row-major, v is 2(M+1) x L row-major */
int ko_build_uv(double weight, const double* profile /*2M+1*/, int L,
                const double* nodes, int modes, double* u, double* v);

/* ---- kron.hpp -------------------------------------------------------- */
/* kron_matvec_shuffle with dense factors (kron.hpp:180-197).
 * factors[p] is rows[p] x cols[p] row-major; q has prod(cols) entries, out
 * prod(rows). *multiplies receives the instrumented multiply count. */
int ko_kron_matvec_shuffle(int d, const int* rows, const int* cols,
                           const double* const* factors, const double* q,
                           double* out, int64_t* multiplies);
int64_t ko_op_count_estimate(int d, const int* rows, const int* cols);

/* ---- parallel.hpp ---------------------------------------------------- */
typedef struct {
    double xi;             /* EwaldConfig.xi */
    int modes;             /* EwaldConfig.modes */
    double center[3];      /* CellGrid.box.center */
    double radius;         /* CellGrid.box.radius */
    int counts[3];         /* CellGrid.counts */
    int order;             /* interpolation order L */
    int dec_modes;         /* SkpDecomposition.modes */
    double correction;     /* SkpDecomposition.correction */
    int nterms;
    const double* term_weights; /* [nterms] */
    const double* profiles;     /* [nterms][3][2M+1] */
    int64_t n;
    const double* pos;     /* [n][3] */
    const double* q;       /* [n] */
    int fuse_terms;
    int threads;
} ko_apply_args;

/* kpme_apply (parallel.hpp:243-290). potentials[n] in global particle
 * order. ledger (nullable) receives 4 int64 per row (rank, step,
 * group_axis, payload) up to ledger_cap rows; *ledger_rows gets the total. */
int ko_kpme_apply(const ko_apply_args* args, double* potentials,
                  int64_t* ledger, int64_t ledger_cap, int64_t* ledger_rows);

/* Stage entry points (same arithmetic as inside ko_kpme_apply). Per-cell
 * grids are [K0*K1*K2][L^3], cells flattened like CellGrid::flatten. */
int ko_interpolate(const ko_apply_args* args, double* phi_cells);
int ko_spkmv_sum(const ko_apply_args* args, const double* phi_cells,
                 double* psi_cells);
int ko_anterpolate(const ko_apply_args* args, const double* psi_cells,
                   double* out);

/* ---- oracle.hpp ------------------------------------------------------ */
/* dense_reciprocal_apply (oracle.hpp:21-58), targets == sources */
int ko_dense_reciprocal_apply(int64_t n, const double* pos, const double* q,
                              double xi, int modes, double* out);

#ifdef __cplusplus
}
#endif
#endif
