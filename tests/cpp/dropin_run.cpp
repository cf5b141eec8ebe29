// Runs config 1 through the C++ drop-in (include/kpme_b200/kpme.hpp) with
// stand-in types that have the reference's member layout, and prints the
// potentials (one per line, %.17g). tests/test_gpu_dropin.py compares them
// with the reference's golden vector.
#include <array>
#include <cmath>
#include <cstdio>
#include <vector>

#include "kpme_b200/kpme.hpp"

namespace ref {
struct VectorXd {  // Eigen-style access, as SkpTerm::profiles (alpha.hpp:69-73)
    std::vector<double> v;
    double operator()(long i) const { return v[i]; }
};
struct EwaldConfig { double xi = 3.0; int modes = 4; };
struct Box3 { std::array<double, 3> center{0.5, 0.5, 0.5}; double radius = 0.5; };
struct CellGrid { Box3 box; std::array<int, 3> counts{8, 8, 8}; };
struct SkpTerm { double weight = 0; std::array<VectorXd, 3> profiles; };
struct SkpDecomposition { int modes = 4; double correction = 0; std::vector<SkpTerm> terms; };
struct PointCloud { std::vector<std::array<double, 3>> positions; };
struct ChargeVector { std::vector<double> values; };
struct KpmeOptions { bool fuse_terms = false; int threads = 1; };
struct LedgerRow { int rank = 0; int step = 0; int group_axis = -1; long long payload = 0; };
struct KpmeResult { std::vector<double> potentials; std::vector<LedgerRow> ledger; };
}  // namespace ref

int main() {
    const int N = 1000, M = 4;
    ref::EwaldConfig cfg;
    ref::CellGrid grid;
    std::vector<double> xyz(3 * N), q(N);
    const double c[3] = {0.5, 0.5, 0.5};
    kpme_sample_cloud(c, 0.5, N, 0, xyz.data(), q.data());
    ref::PointCloud cloud;
    ref::ChargeVector charges;
    for (int i = 0; i < N; ++i) {
        cloud.positions.push_back({xyz[3 * i], xyz[3 * i + 1], xyz[3 * i + 2]});
        charges.values.push_back(i < N / 2 ? 1.0 : -1.0);
    }
    std::vector<double> nodes(801), weights(801);
    int nq = 0;
    double h = 0, e = 0;
    kpme_b200::throw_status(kpme_sinc_rule_for_eps(1e-8, M, 400, &nq, nodes.data(),
                                                   weights.data(), &h, &e));
    const int cnt = 2 * nq + 1;
    const int P = 2 * M + 1;
    std::vector<double> tw(cnt), prof((size_t)cnt * 3 * P);
    ref::SkpDecomposition dec;
    kpme_b200::throw_status(kpme_skp_from_quadrature(cnt, nodes.data(), weights.data(), 1.0,
                                                     3.0 * M * M, cfg.xi, M, tw.data(),
                                                     prof.data(), &dec.correction));
    for (int t = 0; t < cnt; ++t) {
        ref::SkpTerm term;
        term.weight = tw[t];
        for (int a = 0; a < 3; ++a)
            term.profiles[a].v.assign(prof.begin() + ((size_t)t * 3 + a) * P,
                                      prof.begin() + ((size_t)t * 3 + a + 1) * P);
        dec.terms.push_back(term);
    }
    const ref::KpmeResult r =
        kpme_b200::kpme_apply<ref::KpmeResult>(cfg, grid, 4, dec, cloud, charges, ref::KpmeOptions{});
    std::printf("ledger_rows %zu\n", r.ledger.size());
    for (double z : r.potentials) std::printf("%.17g\n", z);
    // error contract: a particle outside the box -> std::invalid_argument
    ref::PointCloud bad = cloud;
    bad.positions[7] = {1.5, 0.5, 0.5};
    try {
        kpme_b200::kpme_apply(cfg, grid, 4, dec, bad, charges, ref::KpmeOptions{});
        std::printf("no_throw\n");
    } catch (const std::invalid_argument& ex) {
        std::printf("invalid_argument %s\n", ex.what());
    }
    return 0;
}
