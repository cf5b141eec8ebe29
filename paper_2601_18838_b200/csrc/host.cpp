// host.cpp -- host-side pieces of the C ABI: error reporting, SKP
// construction (the reference's host code: alpha.hpp:99-212), deterministic
// sampling (geometry.hpp:219-251) and the logical message ledger
// (parallel.hpp:84-145). None of this is on the device path; kpme_apply
// callers normally build the decomposition once, outside the timed call
// (tools/kpme.cpp:64-77).
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <limits>
#include <string>
#include <vector>

#include "internal.h"

namespace kb {
thread_local std::string g_last_error;
}

using kb::Error;

extern "C" const char* kpme_gpu_last_error(void) { return kb::g_last_error.c_str(); }
extern "C" int kpme_gpu_abi_version(void) { return KPME_GPU_ABI_VERSION; }

namespace {

template <class F>
int guarded(F&& f) {
    try {
        f();
        return KPME_GPU_OK;
    } catch (const Error& e) {
        kb::g_last_error = e.what();
        return e.code;
    } catch (const std::exception& e) {
        kb::g_last_error = e.what();
        return KPME_GPU_RUNTIME;
    }
}

// max over integer R in [1, max_arg] of |1/R - sum_l w_l exp(-lambda_l R)|
// (quadrature_max_error, alpha.hpp:99-108)
double max_error(const std::vector<double>& nodes, const std::vector<double>& weights,
                 long long max_arg) {
    double worst = 0.0;
    for (long long r = 1; r <= max_arg; ++r) {
        double s = 0.0;
        for (size_t l = 0; l < nodes.size(); ++l) s += weights[l] * std::exp(-nodes[l] * double(r));
        const double e = std::abs(1.0 / double(r) - s);
        if (worst < e) worst = e;
    }
    return worst;
}

// Sinc rule with step scan (sinc_rule, alpha.hpp:114-151).
int sinc_rule_impl(int n_quad, int modes, std::vector<double>& nodes, std::vector<double>& weights,
                   double* lifting, double* eps) {
    if (n_quad < 1) throw Error(KPME_GPU_INVALID_ARGUMENT, "sinc_rule: n_quad must be >= 1");
    if (modes < 1) throw Error(KPME_GPU_INVALID_ARGUMENT, "sinc_rule: modes must be >= 1");
    const double h_star = M_PI / std::sqrt(2.0 * n_quad + 1.0);
    const long long max_arg = 3LL * modes * modes;
    std::vector<double> tn(2 * n_quad + 1), tw(2 * n_quad + 1);
    double best = std::numeric_limits<double>::infinity(), best_h = 0.0;
    constexpr int kCandidates = 64;
    for (int c = 0; c < kCandidates; ++c) {
        const double t = double(c) / (kCandidates - 1);
        const double h = (h_star / 4.0) * std::pow(16.0, t);
        for (int l = -n_quad; l <= n_quad; ++l) {
            tw[l + n_quad] = h / (1.0 + std::exp(-l * h));
            tn[l + n_quad] = std::log1p(std::exp(l * h));
        }
        const double err = max_error(tn, tw, max_arg);
        if (err < best) {
            best = err;
            best_h = h;
            nodes = tn;
            weights = tw;
        }
    }
    if (nodes.empty()) throw Error(KPME_GPU_NUMERICAL, "sinc_rule: no finite candidate");
    *lifting = best_h;
    *eps = best;
    return 0;
}

}  // namespace

extern "C" int kpme_sinc_rule(int n_quad, int modes, double* nodes, double* weights,
                              double* lifting, double* eps) {
    return guarded([&] {
        std::vector<double> n, w;
        sinc_rule_impl(n_quad, modes, n, w, lifting, eps);
        std::memcpy(nodes, n.data(), sizeof(double) * n.size());
        std::memcpy(weights, w.data(), sizeof(double) * w.size());
    });
}

// sinc_rule_for_eps (alpha.hpp:154-161)
extern "C" int kpme_sinc_rule_for_eps(double eps, int modes, int max_n, int* n_quad,
                                      double* nodes, double* weights, double* lifting,
                                      double* eps_out) {
    return guarded([&] {
        if (!(eps > 0.0))
            throw Error(KPME_GPU_INVALID_ARGUMENT, "sinc_rule_for_eps: eps must be positive");
        for (int n = 1; n <= max_n; ++n) {
            std::vector<double> nd, wt;
            double h, e;
            sinc_rule_impl(n, modes, nd, wt, &h, &e);
            if (e <= eps) {
                *n_quad = n;
                std::memcpy(nodes, nd.data(), sizeof(double) * nd.size());
                std::memcpy(weights, wt.data(), sizeof(double) * wt.size());
                *lifting = h;
                *eps_out = e;
                return;
            }
        }
        throw Error(KPME_GPU_NUMERICAL, "sinc_rule_for_eps: eps not reached within node budget");
    });
}

// skp_from_quadrature (alpha.hpp:165-188)
extern "C" int kpme_skp_from_quadrature(int count, const double* nodes, const double* weights,
                                        double min_arg, double max_arg, double xi, int modes,
                                        double* term_weights, double* profiles,
                                        double* correction) {
    return guarded([&] {
        const int M = modes;
        if (!(xi > 0.0)) throw Error(KPME_GPU_INVALID_ARGUMENT, "EwaldConfig: xi must be positive");
        if (M < 1) throw Error(KPME_GPU_INVALID_ARGUMENT, "EwaldConfig: modes must be >= 1");
        if (!(min_arg <= 1.0 && max_arg >= 3.0 * M * M))
            throw Error(KPME_GPU_INVALID_ARGUMENT,
                        "skp_from_quadrature: rule does not cover arguments [1, 3M^2]");
        const double shift = (M_PI / xi) * (M_PI / xi);
        const int P = 2 * M + 1;
        double c = 0.0;
        for (int l = 0; l < count; ++l) {
            term_weights[l] = weights[l];
            for (int m = -M; m <= M; ++m) {
                const double v = std::exp(-(nodes[l] + shift) * double(m) * double(m));
                for (int a = 0; a < 3; ++a) profiles[((long long)l * 3 + a) * P + m + M] = v;
            }
            c += weights[l];
        }
        *correction = c;
    });
}

// load_tabulated_rule (alpha.hpp:192-212): "count", count lines "node weight",
// trailer "min_arg max_arg eps".
extern "C" int kpme_load_tabulated_rule(const char* path, int cap, int* count, double* nodes,
                                        double* weights, double* min_arg, double* max_arg,
                                        double* eps) {
    return guarded([&] {
        std::ifstream in(path);
        if (!in) throw Error(KPME_GPU_RUNTIME, std::string("load_tabulated_rule: cannot open ") + path);
        int c = 0;
        if (!(in >> c) || c < 1)
            throw Error(KPME_GPU_RUNTIME, "load_tabulated_rule: missing or invalid node count");
        if (c > cap) throw Error(KPME_GPU_INVALID_ARGUMENT, "load_tabulated_rule: capacity too small");
        for (int i = 0; i < c; ++i)
            if (!(in >> nodes[i] >> weights[i]))
                throw Error(KPME_GPU_RUNTIME, "load_tabulated_rule: malformed node line " +
                                                  std::to_string(i + 2));
        if (!(in >> *min_arg >> *max_arg >> *eps))
            throw Error(KPME_GPU_RUNTIME, "load_tabulated_rule: missing trailer line");
        *count = c;
    });
}

// sample_cloud (geometry.hpp:238-251) with splitmix64 SeededUniform (219-233)
extern "C" void kpme_sample_cloud(const double center[3], double radius, int64_t n, uint64_t seed,
                                  double* xyz, double* q) {
    uint64_t st = seed;
    auto next01 = [&st]() {
        uint64_t z = (st += 0x9e3779b97f4a7c15ULL);
        z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
        z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
        z ^= z >> 31;
        return double(z >> 11) * 0x1.0p-53;
    };
    for (int64_t i = 0; i < n; ++i) {
        for (int a = 0; a < 3; ++a) xyz[3 * i + a] = center[a] + radius * (2.0 * next01() - 1.0);
        q[i] = 2.0 * next01() - 1.0;
    }
}

// The logical per-cell ledger of SimulatedComm (parallel.hpp:110-138) as
// kpme_apply produces it: one scalar all-reduce, then per term (unfused) or
// once (fused) three axis reductions p = 2, 1, 0 of 2(M+1) L^2 (x terms).
extern "C" int kpme_gpu_ledger(const kpme_gpu_config* cfg, int64_t* out, int64_t cap,
                               int64_t* rows) {
    return guarded([&] {
        const int64_t ncell = (int64_t)cfg->counts[0] * cfg->counts[1] * cfg->counts[2];
        const int64_t base = 2LL * (cfg->modes + 1) * cfg->order * cfg->order;
        int64_t k = 0;
        auto push = [&](int64_t r, int64_t step, int64_t axis, int64_t payload) {
            if (out && k < cap) {
                out[4 * k] = r;
                out[4 * k + 1] = step;
                out[4 * k + 2] = axis;
                out[4 * k + 3] = payload;
            }
            ++k;
        };
        int step = 0;
        for (int64_t r = 0; r < ncell; ++r) push(r, step, -1, 1);
        ++step;
        if (cfg->nterms > 0) {
            const int blocks = cfg->fuse_terms ? 1 : cfg->nterms;
            const int64_t payload = cfg->fuse_terms ? base * cfg->nterms : base;
            for (int b = 0; b < blocks; ++b)
                for (int p = 2; p >= 0; --p, ++step)
                    for (int64_t r = 0; r < ncell; ++r) push(r, step, p, payload);
        }
        *rows = k;
    });
}

// ---- SVD-kind decompositions (alpha.hpp:42-65, 214-281) -------------------

namespace {

// alpha_weight (alpha.hpp:34-39): exp(-pi^2 |m|^2 / xi^2) / |m|^2, 0 at m = 0.
double alpha_at(double xi, int m0, int m1, int m2) {
    const double r2 = double(m0) * m0 + double(m1) * m1 + double(m2) * m2;
    if (r2 == 0.0) return 0.0;
    const double p = M_PI / xi;
    return std::exp(-p * p * r2) / r2;
}

// Thin SVD a = U diag(s) V^T of a row-major m x n matrix by one-sided
// (Hestenes) Jacobi rotations on the columns of the taller orientation;
// k = min(m, n) singular values, descending. U: m x k, V: n x k, row-major.
// Signs: each pair (U_j, V_j) is flipped so that the largest-magnitude entry
// of V_j is positive (the product U_j s_j V_j^T is sign-free).
void jacobi_svd(int m, int n, const std::vector<double>& a, std::vector<double>& U,
                std::vector<double>& s, std::vector<double>& V) {
    const bool tall = m >= n;
    const int r = tall ? m : n, c = tall ? n : m;  // work on r x c, columns rotated
    std::vector<double> w((size_t)r * c), j((size_t)c * c, 0.0);
    for (int i = 0; i < r; ++i)
        for (int k = 0; k < c; ++k) w[(size_t)i * c + k] = tall ? a[(size_t)i * n + k] : a[(size_t)k * n + i];
    for (int k = 0; k < c; ++k) j[(size_t)k * c + k] = 1.0;
    for (int sweep = 0; sweep < 100; ++sweep) {
        double off = 0.0;
        for (int p = 0; p < c; ++p)
            for (int q = p + 1; q < c; ++q) {
                double al = 0.0, be = 0.0, ga = 0.0;
                for (int i = 0; i < r; ++i) {
                    const double x = w[(size_t)i * c + p], y = w[(size_t)i * c + q];
                    al += x * x;
                    be += y * y;
                    ga += x * y;
                }
                if (ga == 0.0 || al == 0.0 || be == 0.0) continue;
                off = std::max(off, std::abs(ga) / std::sqrt(al * be));
                const double zeta = (be - al) / (2.0 * ga);
                const double t = (zeta >= 0.0 ? 1.0 : -1.0) / (std::abs(zeta) + std::sqrt(1.0 + zeta * zeta));
                const double cs = 1.0 / std::sqrt(1.0 + t * t), sn = cs * t;
                for (int i = 0; i < r; ++i) {
                    double& x = w[(size_t)i * c + p];
                    double& y = w[(size_t)i * c + q];
                    const double xo = x, yo = y;
                    x = cs * xo - sn * yo;
                    y = sn * xo + cs * yo;
                }
                for (int i = 0; i < c; ++i) {
                    double& x = j[(size_t)i * c + p];
                    double& y = j[(size_t)i * c + q];
                    const double xo = x, yo = y;
                    x = cs * xo - sn * yo;
                    y = sn * xo + cs * yo;
                }
            }
        if (off < 1e-15) break;
    }
    // column norms = singular values; Q = w / s (r x c), J (c x c)
    std::vector<double> sv(c);
    for (int k = 0; k < c; ++k) {
        double t = 0.0;
        for (int i = 0; i < r; ++i) t += w[(size_t)i * c + k] * w[(size_t)i * c + k];
        sv[k] = std::sqrt(t);
    }
    std::vector<int> order(c);
    for (int k = 0; k < c; ++k) order[k] = k;
    std::stable_sort(order.begin(), order.end(), [&](int x, int y) { return sv[x] > sv[y]; });
    // tall: a = Q S J^T -> U = Q, V = J; wide: a^T = Q S J^T -> U = J, V = Q
    U.assign((size_t)m * c, 0.0);
    V.assign((size_t)n * c, 0.0);
    s.assign(c, 0.0);
    for (int kk = 0; kk < c; ++kk) {
        const int k = order[kk];
        s[kk] = sv[k];
        std::vector<double> qk(r), jk(c);
        for (int i = 0; i < r; ++i) qk[i] = sv[k] > 0.0 ? w[(size_t)i * c + k] / sv[k] : 0.0;
        for (int i = 0; i < c; ++i) jk[i] = j[(size_t)i * c + k];
        const std::vector<double>& uk = tall ? qk : jk;
        const std::vector<double>& vk = tall ? jk : qk;
        int big = 0;
        for (int i = 1; i < n; ++i)
            if (std::abs(vk[i]) > std::abs(vk[big])) big = i;
        const double sg = vk[big] < 0.0 ? -1.0 : 1.0;
        for (int i = 0; i < m; ++i) U[(size_t)i * c + kk] = sg * uk[i];
        for (int i = 0; i < n; ++i) V[(size_t)i * c + kk] = sg * vk[i];
    }
}

}  // namespace

// assemble_alpha (alpha.hpp:54-65): entries[((m0+M) n + (m1+M)) n + (m2+M)].
extern "C" int kpme_assemble_alpha(double xi, int modes, double* entries) {
    return guarded([&] {
        if (!(xi > 0.0)) throw Error(KPME_GPU_INVALID_ARGUMENT, "EwaldConfig: xi must be positive");
        if (modes < 1) throw Error(KPME_GPU_INVALID_ARGUMENT, "EwaldConfig: modes must be >= 1");
        if (!entries) throw Error(KPME_GPU_INVALID_ARGUMENT, "kpme_assemble_alpha: null output");
        const int M = modes, n = 2 * M + 1;
        for (int m0 = -M; m0 <= M; ++m0)
            for (int m1 = -M; m1 <= M; ++m1)
                for (int m2 = -M; m2 <= M; ++m2)
                    entries[((size_t)(m0 + M) * n + (m1 + M)) * n + (m2 + M)] = alpha_at(xi, m0, m1, m2);
    });
}

// nkpa_svd (alpha.hpp:225-281): two nested truncated SVDs -- the unfolding
// with axis-0 rows, then each kept right singular vector unfolded with axis-1
// rows -- keeping singular values > tol * s_max. Terms: weight s_i s_ij,
// profiles (u_i, u_ij, v_ij) over m = -M..M; correction 0.
extern "C" int kpme_nkpa_svd(int modes, const double* alpha, double tol_outer, double tol_inner,
                             int cap, int* nterms, double* term_weights, double* profiles,
                             double* error_bound) {
    return guarded([&] {
        if (tol_inner > tol_outer)
            throw Error(KPME_GPU_INVALID_ARGUMENT, "nkpa_svd: tol_inner must be <= tol_outer");
        if (modes < 1 || !alpha || !nterms)
            throw Error(KPME_GPU_INVALID_ARGUMENT, "kpme_nkpa_svd: bad argument");
        const int n = 2 * modes + 1;
        std::vector<double> outer(alpha, alpha + (size_t)n * n * n);  // matricize axis 0: n x n^2
        std::vector<double> U0, s0, V0;
        jacobi_svd(n, n * n, outer, U0, s0, V0);
        double sum0 = 0.0;
        for (double v : s0) sum0 += v;
        if (!std::isfinite(sum0))
            throw Error(KPME_GPU_NUMERICAL, "nkpa_svd: outer SVD produced non-finite values");
        const int k0 = (int)s0.size();
        const double s0max = k0 ? s0[0] : 0.0;
        double bound = 0.0, tail0 = 0.0;
        int count = 0;
        for (int i = 0; i < k0; ++i) {
            if (s0max == 0.0 || s0[i] <= tol_outer * s0max) {
                tail0 += s0[i] * s0[i];
                continue;
            }
            std::vector<double> inner((size_t)n * n);  // matricize(w, {n, n}, 0)
            for (int e = 0; e < n * n; ++e) inner[e] = V0[(size_t)e * k0 + i];
            std::vector<double> U1, s1, V1;
            jacobi_svd(n, n, inner, U1, s1, V1);
            double sum1 = 0.0;
            for (double v : s1) sum1 += v;
            if (!std::isfinite(sum1))
                throw Error(KPME_GPU_NUMERICAL, "nkpa_svd: inner SVD produced non-finite values");
            const int k1 = (int)s1.size();
            const double s1max = k1 ? s1[0] : 0.0;
            double tail1 = 0.0;
            for (int jj = 0; jj < k1; ++jj) {
                if (s1max == 0.0 || s1[jj] <= tol_inner * s1max) {
                    tail1 += s1[jj] * s1[jj];
                    continue;
                }
                if (count < cap && term_weights && profiles) {
                    term_weights[count] = s0[i] * s1[jj];
                    double* p = profiles + (size_t)count * 3 * n;
                    for (int m = 0; m < n; ++m) {
                        p[m] = U0[(size_t)m * k0 + i];
                        p[n + m] = U1[(size_t)m * k1 + jj];
                        p[2 * n + m] = V1[(size_t)m * k1 + jj];
                    }
                }
                ++count;
            }
            bound += s0[i] * std::sqrt(tail1);
        }
        bound += std::sqrt(tail0);
        *nterms = count;
        if (error_bound) *error_bound = bound;
        if (count > cap && term_weights)
            throw Error(KPME_GPU_INVALID_ARGUMENT, "kpme_nkpa_svd: more terms than cap (" +
                                                       std::to_string(count) + ")");
    });
}
