// kpme_b200/kpme.hpp -- C++ drop-in for kpme::kpme_apply on B200.
//
// Header-only wrapper over the C ABI (include/kpme_gpu.h). The function
// templates accept the reference's own argument types
// (kpme::EwaldConfig, kpme::CellGrid, kpme::SkpDecomposition with its Eigen
// profiles, kpme::PointCloud, kpme::ChargeVector, kpme::KpmeOptions from
// /root/reference/proj/include/kpme/) -- or any types with the same members --
// so a caller switches by replacing `kpme::kpme_apply(...)` with
// `kpme_b200::kpme_apply(...)`. Errors are rethrown as the
// reference's exception types: std::invalid_argument, std::runtime_error and
// (via NumericalError) kpme::numerical_error.
#pragma once

#include <array>
#include <cstdint>
#include <cstdlib>
#include <stdexcept>
#include <string>
#include <type_traits>
#include <utility>
#include <vector>

#include "kpme_gpu.h"

namespace kpme_b200 {

struct numerical_error : std::runtime_error {
    using std::runtime_error::runtime_error;
};

struct LedgerRow {  // parallel.hpp:84-89
    int rank = 0;
    int step = 0;
    int group_axis = -1;
    long long payload = 0;
};

struct KpmeResult {  // parallel.hpp:235-238
    std::vector<double> potentials;
    std::vector<LedgerRow> ledger;
};

struct GpuOptions {
    int device = 0;
    int formulation = KPME_GPU_FORM_AUTO;
    bool ledger = true;  // synthesise KpmeResult::ledger
    // More than one device: one process drives them all (a multi-device plan:
    // cell blocks per device, partial cores summed over NVLink peer memory or
    // NCCL). Empty: `device` alone.
    std::vector<int> devices;

    // Defaults for calls that carry no GPU options (the reference signature):
    // KPME_GPU_DEVICES="0,1,2,3" (a device list) or KPME_GPU_DEVICE=<n>.
    static GpuOptions from_env() {
        GpuOptions g;
        if (const char* e = std::getenv("KPME_GPU_DEVICE")) g.device = std::atoi(e);
        if (const char* e = std::getenv("KPME_GPU_DEVICES")) {
            const std::string s(e);
            std::size_t i = 0;
            while (i < s.size()) {
                std::size_t j = s.find(',', i);
                if (j == std::string::npos) j = s.size();
                if (j > i) g.devices.push_back(std::atoi(s.substr(i, j - i).c_str()));
                i = j + 1;
            }
            if (!g.devices.empty()) g.device = g.devices[0];
        }
        return g;
    }
};

// KpmeOptions defaults (parallel.hpp:230-233) for calls that omit them.
struct DefaultOptions {
    bool fuse_terms = false;
    int threads = 1;
};

template <class NumericalError = numerical_error>
inline void throw_status(int st) {
    if (st == KPME_GPU_OK) return;
    const std::string msg = kpme_gpu_last_error();
    if (st == KPME_GPU_INVALID_ARGUMENT) throw std::invalid_argument(msg);
    if (st == KPME_GPU_NUMERICAL) throw NumericalError(msg);
    throw std::runtime_error(msg);
}

namespace detail {
// profile element access: Eigen's v(i) or a container's v[i]
template <class V>
auto at(const V& v, int i, int) -> decltype(double(v(i))) {
    return double(v(i));
}
template <class V>
auto at(const V& v, int i, long) -> decltype(double(v[i])) {
    return double(v[i]);
}

// Flattened decomposition in the ABI layout [nterms][3][2M+1].
struct Flat {
    std::vector<double> weights, profiles;
};
template <class Dec>
Flat flatten_dec(const Dec& dec) {
    Flat f;
    const int P = 2 * dec.modes + 1;
    for (const auto& t : dec.terms) {
        f.weights.push_back(double(t.weight));
        for (int a = 0; a < 3; ++a)
            for (int m = 0; m < P; ++m) f.profiles.push_back(at(t.profiles[a], m, 0));
    }
    return f;
}

template <class Cfg, class Grid, class Dec, class Opt>
kpme_gpu_config make_config(const Cfg& cfg, const Grid& grid, int order, const Dec& dec,
                            const Opt& opt, const Flat& f, const GpuOptions& gpu) {
    kpme_gpu_config c{};
    c.xi = cfg.xi;
    c.modes = cfg.modes;
    for (int a = 0; a < 3; ++a) {
        c.center[a] = grid.box.center[a];
        c.counts[a] = grid.counts[a];
    }
    c.radius = grid.box.radius;
    c.order = order;
    c.dec_modes = dec.modes;
    c.correction = dec.correction;
    c.nterms = int(f.weights.size());
    c.term_weights = f.weights.data();
    c.profiles = f.profiles.data();
    c.fuse_terms = opt.fuse_terms ? 1 : 0;
    c.threads = opt.threads;
    c.device = gpu.devices.empty() ? gpu.device : gpu.devices[0];
    c.formulation = gpu.formulation;
    c.ndevices = int(gpu.devices.size());
    c.devices = gpu.devices.empty() ? nullptr : gpu.devices.data();
    return c;
}

// PointCloud::positions as double[n][3]: the reference's
// std::vector<std::array<double, 3>> already has that layout, so it is passed
// through without a copy; other position types are copied once.
template <class Cloud>
const double* positions_aos(const Cloud& cloud, std::vector<double>& tmp) {
    using P = std::decay_t<decltype(cloud.positions[0])>;
    const std::size_t n = cloud.positions.size();
    if constexpr (std::is_same_v<P, std::array<double, 3>>) {
        static_assert(sizeof(P) == 3 * sizeof(double), "std::array<double, 3> is padded");
        return n ? cloud.positions[0].data() : nullptr;
    } else {
        tmp.resize(3 * n);
        for (std::size_t i = 0; i < n; ++i)
            for (int a = 0; a < 3; ++a) tmp[3 * i + a] = double(cloud.positions[i][a]);
        return tmp.data();
    }
}

template <class Row>
std::vector<Row> ledger(const kpme_gpu_config& c) {
    int64_t rows = 0;
    throw_status(kpme_gpu_ledger(&c, nullptr, 0, &rows));
    std::vector<int64_t> raw(4 * rows);
    throw_status(kpme_gpu_ledger(&c, raw.data(), rows, &rows));
    std::vector<Row> out;
    out.reserve(rows);
    for (int64_t i = 0; i < rows; ++i)
        out.push_back(Row{int(raw[4 * i]), int(raw[4 * i + 1]), int(raw[4 * i + 2]),
                          (long long)raw[4 * i + 3]});
    return out;
}
}  // namespace detail

// kpme_apply (parallel.hpp:243-290). Result defaults to kpme_b200::KpmeResult;
// pass kpme::KpmeResult to get the reference's own result type. The one-shot
// call reuses a cached plan for repeated configurations (kpme_gpu_apply).
template <class Result = KpmeResult, class NumericalError = numerical_error, class Cfg,
          class Grid, class Dec, class Cloud, class Charges, class Opt>
Result kpme_apply(const Cfg& cfg, const Grid& grid, int order, const Dec& dec, const Cloud& cloud,
                  const Charges& q, const Opt& opt, const GpuOptions& gpu = GpuOptions::from_env()) {
    if (dec.modes != cfg.modes)
        throw std::invalid_argument("kpme_apply: decomposition mode bound mismatch");
    const std::size_t n = cloud.positions.size();
    if (q.values.size() != n) throw std::invalid_argument("interpolate: charge count mismatch");
    const detail::Flat f = detail::flatten_dec(dec);
    const kpme_gpu_config c = detail::make_config(cfg, grid, order, dec, opt, f, gpu);
    std::vector<double> tmp;
    const double* xyz = detail::positions_aos(cloud, tmp);
    Result r;
    r.potentials.assign(n, 0.0);
    throw_status<NumericalError>(
        kpme_gpu_apply(&c, int64_t(n), xyz, q.values.data(), r.potentials.data()));
    if (gpu.ledger)
        r.ledger = detail::ledger<typename std::decay_t<decltype(r.ledger)>::value_type>(c);
    return r;
}

// The reference's six-argument form (KpmeOptions defaulted, parallel.hpp:
// 243-246): GPU options from the environment (GpuOptions::from_env).
template <class Result = KpmeResult, class NumericalError = numerical_error, class Cfg,
          class Grid, class Dec, class Cloud, class Charges>
Result kpme_apply(const Cfg& cfg, const Grid& grid, int order, const Dec& dec, const Cloud& cloud,
                  const Charges& q) {
    return kpme_apply<Result, NumericalError>(cfg, grid, order, dec, cloud, q, DefaultOptions{},
                                              GpuOptions::from_env());
}

// Steady-state plan: factor tables built once, device buffers reused.
class Plan {
  public:
    template <class Cfg, class Grid, class Dec, class Opt>
    Plan(const Cfg& cfg, const Grid& grid, int order, const Dec& dec, const Opt& opt,
         int64_t max_particles, const GpuOptions& gpu = {}) {
        const detail::Flat f = detail::flatten_dec(dec);
        const kpme_gpu_config c = detail::make_config(cfg, grid, order, dec, opt, f, gpu);
        throw_status(kpme_gpu_plan_create(&c, max_particles, &plan_));
    }
    Plan(const Plan&) = delete;
    Plan& operator=(const Plan&) = delete;
    ~Plan() { kpme_gpu_plan_destroy(plan_); }

    // host buffers: xyz[n][3], q[n] -> potentials[n]
    void apply(int64_t n, const double* xyz, const double* q, double* potentials) {
        throw_status(kpme_gpu_plan_execute(plan_, n, xyz, q, potentials));
    }
    // device buffers, stream-ordered
    void apply_device(int64_t n, const double* d_xyz, const double* d_q, double* d_out,
                      bool defer_checks = false) {
        throw_status(kpme_gpu_plan_execute_device(plan_, n, d_xyz, d_q, d_out,
                                                  defer_checks ? KPME_GPU_DEFER_CHECKS : 0));
    }
    void set_stream(void* stream) { throw_status(kpme_gpu_plan_set_stream(plan_, stream)); }
    kpme_gpu_plan handle() const { return plan_; }

  private:
    kpme_gpu_plan plan_ = nullptr;
};

}  // namespace kpme_b200
