// kpme_ref_capi.cpp -- TEST INFRASTRUCTURE ONLY.
//
// Thin extern "C" shim over the reference's own, unmodified headers
// (/root/reference/proj/include/kpme/*.hpp, included by path at build time,
// never copied). Built by oracle/ref/Makefile into oracle/_ref/libkpme_ref.so
// against the clean-room Eigen subset in oracle/ref/eigen_shim. Used to pin
// the C oracle (tests/test_oracle_pins.py), to generate the committed golden
// vectors (tests/golden/gen_golden.py) and as the reference CPU arm of
// bench.py (--impl reference / cpu_baseline kind "reference").
#include "kpme/alpha.hpp"
#include "kpme/geometry.hpp"
#include "kpme/interpolation.hpp"
#include "kpme/kron.hpp"
#include "kpme/oracle.hpp"
#include "kpme/parallel.hpp"
#include "kpme/symfourier.hpp"

#include "../kpme_oracle.h"  // for the shared ko_apply_args layout only

#include <cstdio>
#include <cstring>
#include <exception>
#include <fstream>
#include <string>

using namespace kpme;

namespace {
thread_local std::string g_err;

template <class F>
int guarded(F&& f) {
    try {
        f();
        return 0;
    } catch (const std::invalid_argument& e) {
        g_err = e.what();
        return 1;
    } catch (const numerical_error& e) {
        g_err = e.what();
        return 3;
    } catch (const std::runtime_error& e) {
        g_err = e.what();
        return 2;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 2;
    }
}

SkpDecomposition make_dec(const ko_apply_args* a) {
    SkpDecomposition dec;
    dec.kind = SkpKind::sinc;
    dec.modes = a->dec_modes;
    dec.correction = a->correction;
    const int P = 2 * a->dec_modes + 1;
    for (int t = 0; t < a->nterms; ++t) {
        SkpTerm term;
        term.weight = a->term_weights[t];
        for (int ax = 0; ax < 3; ++ax) {
            term.profiles[ax] = Eigen::VectorXd(P);
            for (int m = 0; m < P; ++m)
                term.profiles[ax](m) = a->profiles[(std::int64_t(t) * 3 + ax) * P + m];
        }
        dec.terms.push_back(std::move(term));
    }
    return dec;
}

PointCloud make_cloud(std::int64_t n, const double* pos) {
    PointCloud c;
    c.positions.resize(n);
    for (std::int64_t i = 0; i < n; ++i)
        c.positions[i] = {pos[3 * i], pos[3 * i + 1], pos[3 * i + 2]};
    return c;
}

CellGrid make_grid(const ko_apply_args* a) {
    return build_cell_grid(Box3({a->center[0], a->center[1], a->center[2]}, a->radius),
                           {a->counts[0], a->counts[1], a->counts[2]});
}
}  // namespace

extern "C" {

const char* kr_last_error() { return g_err.c_str(); }

void kr_sample_cloud(const double center[3], double radius, std::int64_t n,
                     std::uint64_t seed, double* pos, double* q) {
    const CloudData d = sample_cloud(Box3({center[0], center[1], center[2]}, radius),
                                     std::size_t(n), seed);
    for (std::int64_t i = 0; i < n; ++i) {
        for (int a = 0; a < 3; ++a) pos[3 * i + a] = d.cloud.positions[i][a];
        q[i] = d.charges.values[i];
    }
}

int kr_assign_particles(const double center[3], double radius, const int counts[3],
                        std::int64_t n, const double* pos, std::int32_t* perm,
                        std::int32_t* cell_start) {
    return guarded([&] {
        const CellGrid grid = build_cell_grid(
            Box3({center[0], center[1], center[2]}, radius), {counts[0], counts[1], counts[2]});
        const Partition part = assign_particles(grid, make_cloud(n, pos));
        std::int64_t k = 0;
        cell_start[0] = 0;
        for (std::size_t c = 0; c < part.members.size(); ++c) {
            for (int p : part.members[c]) perm[k++] = p;
            cell_start[c + 1] = std::int32_t(k);
        }
    });
}

double kr_alpha_weight(double xi, int m0, int m1, int m2) {
    return alpha_weight(EwaldConfig(xi, 1), m0, m1, m2);
}

int kr_sinc_rule(int n_quad, int modes, double* nodes, double* weights, double* lifting,
                 double* eps) {
    return guarded([&] {
        const QuadratureRule r = sinc_rule(n_quad, modes);
        std::memcpy(nodes, r.nodes.data(), sizeof(double) * r.nodes.size());
        std::memcpy(weights, r.weights.data(), sizeof(double) * r.weights.size());
        *lifting = r.lifting;
        *eps = r.eps;
    });
}

int kr_sinc_rule_for_eps(double eps, int modes, int max_n, int* n_quad, double* nodes,
                         double* weights, double* lifting, double* eps_out) {
    return guarded([&] {
        const QuadratureRule r = sinc_rule_for_eps(eps, modes, max_n);
        *n_quad = r.half_width;
        std::memcpy(nodes, r.nodes.data(), sizeof(double) * r.nodes.size());
        std::memcpy(weights, r.weights.data(), sizeof(double) * r.weights.size());
        *lifting = r.lifting;
        *eps_out = r.eps;
    });
}

int kr_skp_from_quadrature(int count, const double* nodes, const double* weights,
                           double min_arg, double max_arg, double xi, int modes,
                           double* term_weights, double* profiles, double* correction) {
    return guarded([&] {
        QuadratureRule rule;
        rule.nodes.assign(nodes, nodes + count);
        rule.weights.assign(weights, weights + count);
        rule.min_arg = min_arg;
        rule.max_arg = max_arg;
        const SkpDecomposition dec = skp_from_quadrature(rule, EwaldConfig(xi, modes));
        const int P = 2 * modes + 1;
        for (std::size_t t = 0; t < dec.terms.size(); ++t) {
            term_weights[t] = dec.terms[t].weight;
            for (int ax = 0; ax < 3; ++ax)
                for (int m = 0; m < P; ++m)
                    profiles[(std::int64_t(t) * 3 + ax) * P + m] = dec.terms[t].profiles[ax](m);
        }
        *correction = dec.correction;
    });
}

int kr_load_tabulated_rule(const char* path, int cap, int* count, double* nodes,
                           double* weights, double* min_arg, double* max_arg, double* eps) {
    return guarded([&] {
        const QuadratureRule r = load_tabulated_rule(std::string(path));
        if (int(r.nodes.size()) > cap) throw std::invalid_argument("capacity");
        *count = int(r.nodes.size());
        std::memcpy(nodes, r.nodes.data(), sizeof(double) * r.nodes.size());
        std::memcpy(weights, r.weights.data(), sizeof(double) * r.weights.size());
        *min_arg = r.min_arg;
        *max_arg = r.max_arg;
        *eps = r.eps;
    });
}

long long kr_optimal_term_lower_bound(double eps) { return optimal_term_lower_bound(eps); }

int kr_lagrange_weights_1d(int order, double a, double b, double y, double* w) {
    return guarded([&] {
        const Eigen::VectorXd v = lagrange_weights_1d(order, a, b, y);
        for (int k = 0; k < order; ++k) w[k] = v(k);
    });
}

int kr_build_w(int m, int npts, const double* pts, double* w) {
    return guarded([&] {
        const Eigen::MatrixXd b = build_w(m, std::vector<double>(pts, pts + npts));
        for (int j = 0; j < npts; ++j) {
            w[j] = b(0, j);
            w[npts + j] = b(1, j);
        }
    });
}

int kr_build_uv(double weight, const double* profile, int L, const double* nodes,
                int modes, double* u, double* v) {
    return guarded([&] {
        SkpTerm term;
        term.weight = weight;
        const int P = 2 * modes + 1;
        for (int ax = 0; ax < 3; ++ax) {
            term.profiles[ax] = Eigen::VectorXd(P);
            for (int m = 0; m < P; ++m) term.profiles[ax](m) = profile[m];
        }
        const std::vector<double> nd(nodes, nodes + L);
        const AxisFactorPair pr = build_uv(term, 0, nd, nd, modes);
        const int R = 2 * (modes + 1);
        for (int j = 0; j < L; ++j)
            for (int r = 0; r < R; ++r) {
                u[j * R + r] = pr.u(j, r);
                v[r * L + j] = pr.v(r, j);
            }
    });
}

int kr_kron_matvec_shuffle(int d, const int* rows, const int* cols,
                           const double* const* factors, const double* q, double* out,
                           long long* multiplies) {
    return guarded([&] {
        KronOperand op;
        long long total = 1;
        for (int p = 0; p < d; ++p) {
            Eigen::MatrixXd f(rows[p], cols[p]);
            for (int i = 0; i < rows[p]; ++i)
                for (int j = 0; j < cols[p]; ++j) f(i, j) = factors[p][i * cols[p] + j];
            op.factors.emplace_back(f);
            total *= cols[p];
        }
        Eigen::VectorXd v(total);
        for (long long i = 0; i < total; ++i) v(i) = q[i];
        long long count = 0;
        const Eigen::VectorXd r = kron_matvec_shuffle(op, v, &count);
        for (Eigen::Index i = 0; i < r.size(); ++i) out[i] = r(i);
        if (multiplies) *multiplies = count;
    });
}

long long kr_op_count_estimate(int d, const int* rows, const int* cols) {
    KronOperand op;
    for (int p = 0; p < d; ++p) op.factors.emplace_back(Eigen::MatrixXd(rows[p], cols[p]));
    return op_count_estimate(op);
}

int kr_kpme_apply(const ko_apply_args* a, double* potentials, std::int64_t* ledger,
                  std::int64_t ledger_cap, std::int64_t* ledger_rows) {
    return guarded([&] {
        const EwaldConfig cfg(a->xi, a->modes);
        const CellGrid grid = make_grid(a);
        const SkpDecomposition dec = make_dec(a);
        ChargeVector q;
        q.values.assign(a->q, a->q + a->n);
        KpmeOptions opt;
        opt.fuse_terms = a->fuse_terms != 0;
        opt.threads = a->threads;
        const KpmeResult r =
            kpme_apply(cfg, grid, a->order, dec, make_cloud(a->n, a->pos), q, opt);
        std::memcpy(potentials, r.potentials.data(), sizeof(double) * r.potentials.size());
        if (ledger_rows) *ledger_rows = std::int64_t(r.ledger.size());
        if (ledger)
            for (std::size_t i = 0; i < r.ledger.size() && std::int64_t(i) < ledger_cap; ++i) {
                ledger[4 * i + 0] = r.ledger[i].rank;
                ledger[4 * i + 1] = r.ledger[i].step;
                ledger[4 * i + 2] = r.ledger[i].group_axis;
                ledger[4 * i + 3] = r.ledger[i].payload;
            }
    });
}

// Stage entry points built from the same reference objects kpme_apply uses.
int kr_interpolate(const ko_apply_args* a, double* phi_cells) {
    return guarded([&] {
        const CellGrid grid = make_grid(a);
        const PointCloud cloud = make_cloud(a->n, a->pos);
        const Partition part = assign_particles(grid, cloud);
        const InterpOperator op(grid, part, cloud, a->order);
        ChargeVector q;
        q.values.assign(a->q, a->q + a->n);
        const std::vector<Eigen::VectorXd> phi = op.interpolate(q);
        const long long g3 = op.grid_size();
        for (std::size_t c = 0; c < phi.size(); ++c)
            std::memcpy(phi_cells + c * g3, phi[c].data(), sizeof(double) * g3);
    });
}

int kr_anterpolate(const ko_apply_args* a, const double* psi_cells, double* out) {
    return guarded([&] {
        const CellGrid grid = make_grid(a);
        const PointCloud cloud = make_cloud(a->n, a->pos);
        const Partition part = assign_particles(grid, cloud);
        const InterpOperator op(grid, part, cloud, a->order);
        const long long g3 = op.grid_size();
        std::vector<Eigen::VectorXd> psi(grid.cell_count(), Eigen::VectorXd(g3));
        for (int c = 0; c < grid.cell_count(); ++c)
            std::memcpy(psi[c].data(), psi_cells + c * g3, sizeof(double) * g3);
        const std::vector<double> z = op.anterpolate(psi);
        std::memcpy(out, z.data(), sizeof(double) * z.size());
    });
}

int kr_spkmv_sum(const ko_apply_args* a, const double* phi_cells, double* psi_cells) {
    return guarded([&] {
        const CellGrid grid = make_grid(a);
        const SkpDecomposition dec = make_dec(a);
        SimulatedComm comm(RankGrid(grid.counts), a->threads);
        const int n = comm.grid().size();
        const int order = a->order;
        const long long g3 = static_cast<long long>(order) * order * order;
        // factor loop exactly as kpme_apply (parallel.hpp:261-279)
        std::vector<std::vector<AxisSplitFactors>> terms(dec.terms.size(),
                                                         std::vector<AxisSplitFactors>(n));
        for (int r = 0; r < n; ++r) {
            const std::array<int, 3> cell = comm.grid().unflatten(r);
            std::array<std::vector<double>, 3> nodes;
            for (int ax = 0; ax < 3; ++ax) {
                nodes[ax] = grid.axis_nodes(ax, cell[ax], order);
                for (double& x : nodes[ax]) x -= grid.box.center[ax];
            }
            for (std::size_t t = 0; t < dec.terms.size(); ++t)
                for (int ax = 0; ax < 3; ++ax) {
                    AxisFactorPair pair =
                        build_uv(dec.terms[t], ax, nodes[ax], nodes[ax], a->modes);
                    terms[t][r].u[ax] = std::move(pair.u);
                    terms[t][r].v[ax] = std::move(pair.v);
                }
        }
        std::vector<Eigen::VectorXd> phi(n, Eigen::VectorXd(g3));
        for (int c = 0; c < n; ++c) std::memcpy(phi[c].data(), phi_cells + c * g3, sizeof(double) * g3);
        const std::vector<Eigen::VectorXd> psi = spkmv_sum(comm, terms, phi, order, a->fuse_terms != 0);
        for (int c = 0; c < n; ++c) std::memcpy(psi_cells + c * g3, psi[c].data(), sizeof(double) * g3);
    });
}

int kr_dense_reciprocal_apply(std::int64_t n, const double* pos, const double* q, double xi,
                              int modes, double* out) {
    return guarded([&] {
        const PointCloud c = make_cloud(n, pos);
        const std::vector<double> z = dense_reciprocal_apply(
            c.positions, c.positions, std::vector<double>(q, q + n), EwaldConfig(xi, modes));
        std::memcpy(out, z.data(), sizeof(double) * z.size());
    });
}

// assemble_alpha (alpha.hpp:54-65) and nkpa_svd (alpha.hpp:225-281): the
// SVD-kind decomposition the GPU library's kpme_nkpa_svd is pinned against.
int kr_assemble_alpha(double xi, int modes, double* entries) {
    return guarded([&] {
        const AlphaVector a = assemble_alpha(EwaldConfig(xi, modes));
        for (Eigen::Index i = 0; i < a.entries.size(); ++i) entries[i] = a.entries(i);
    });
}

int kr_nkpa_svd(int modes, const double* alpha, double tol_outer, double tol_inner, int cap,
                int* nterms, double* term_weights, double* profiles, double* error_bound) {
    return guarded([&] {
        const int n = 2 * modes + 1;
        AlphaVector a;
        a.modes = modes;
        a.entries = Eigen::VectorXd(std::int64_t(n) * n * n);
        for (std::int64_t i = 0; i < std::int64_t(n) * n * n; ++i) a.entries(i) = alpha[i];
        double bound = 0.0;
        const SkpDecomposition dec = nkpa_svd(a, tol_outer, tol_inner, &bound);
        *nterms = int(dec.terms.size());
        if (error_bound) *error_bound = bound;
        for (int t = 0; t < *nterms && t < cap; ++t) {
            term_weights[t] = dec.terms[t].weight;
            for (int ax = 0; ax < 3; ++ax)
                for (int m = 0; m < n; ++m)
                    profiles[(std::int64_t(t) * 3 + ax) * n + m] = dec.terms[t].profiles[ax](m);
        }
    });
}

}  // extern "C"
