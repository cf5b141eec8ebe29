// kpme_b200/reroute.hpp -- route the reference's kpme::kpme_apply to the GPU
// without touching the caller's source.
//
// Force-include this header ahead of a translation unit that includes the
// reference's <kpme/parallel.hpp> (g++ -include kpme_b200/reroute.hpp, with
// the reference's include directory on the path). The reference's own
// definition (parallel.hpp:243-290) is compiled under the name
// kpme_apply_reference, and kpme::kpme_apply -- same signature, same default
// KpmeOptions, same result and exception types -- forwards to
// kpme_b200::kpme_apply (C ABI, libkpme_b200.so). GPU options come from the
// environment (KPME_GPU_DEVICE / KPME_GPU_DEVICES, GpuOptions::from_env).
// tests/test_gpu_dropin.py builds the reference's unmodified acceptance.cpp
// this way and runs its eight criteria on the B200.
#pragma once

#define kpme_apply kpme_apply_reference
#include <kpme/parallel.hpp>
#undef kpme_apply

#include "kpme_b200/kpme.hpp"

namespace kpme {
inline KpmeResult kpme_apply(const EwaldConfig& cfg, const CellGrid& grid, int order,
                             const SkpDecomposition& dec, const PointCloud& cloud,
                             const ChargeVector& q, const KpmeOptions& opt = {}) {
    return kpme_b200::kpme_apply<KpmeResult, numerical_error>(cfg, grid, order, dec, cloud, q, opt,
                                                             kpme_b200::GpuOptions::from_env());
}
}  // namespace kpme
