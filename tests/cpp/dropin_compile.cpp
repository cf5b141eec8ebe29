// Instantiates include/kpme_b200/kpme.hpp with stand-ins that have the
// reference's member layout (geometry.hpp, alpha.hpp, parallel.hpp), incl. an
// Eigen-style profile type accessed with operator().
#include <array>
#include <vector>

#include "kpme_b200/kpme.hpp"

namespace ref {
struct VectorXd {
    std::vector<double> v;
    double operator()(long i) const { return v[i]; }
};
struct EwaldConfig { double xi = 3.0; int modes = 4; };
struct Box3 { std::array<double, 3> center{}; double radius = 0.5; };
struct CellGrid { Box3 box; std::array<int, 3> counts{1, 1, 1}; };
struct SkpTerm { double weight = 0; std::array<VectorXd, 3> profiles; };
struct SkpDecomposition { int modes = 4; double correction = 0; std::vector<SkpTerm> terms; };
struct PointCloud { std::vector<std::array<double, 3>> positions; };
struct ChargeVector { std::vector<double> values; };
struct KpmeOptions { bool fuse_terms = false; int threads = 1; };
struct LedgerRow { int rank = 0; int step = 0; int group_axis = -1; long long payload = 0; };
struct KpmeResult { std::vector<double> potentials; std::vector<LedgerRow> ledger; };
}  // namespace ref

ref::KpmeResult run(const ref::EwaldConfig& c, const ref::CellGrid& g,
                    const ref::SkpDecomposition& d, const ref::PointCloud& p,
                    const ref::ChargeVector& q) {
    auto a = kpme_b200::kpme_apply(c, g, 4, d, p, q, ref::KpmeOptions{});
    (void)a;
    // the reference's six-argument call form (KpmeOptions defaulted)
    auto b = kpme_b200::kpme_apply<ref::KpmeResult>(c, g, 4, d, p, q);
    (void)b;
    kpme_b200::GpuOptions multi;
    multi.devices = {0, 1, 2, 3};
    auto m = kpme_b200::kpme_apply(c, g, 4, d, p, q, ref::KpmeOptions{}, multi);
    (void)m;
    kpme_b200::Plan plan(c, g, 4, d, ref::KpmeOptions{}, 16);
    return kpme_b200::kpme_apply<ref::KpmeResult>(c, g, 4, d, p, q, ref::KpmeOptions{});
}
