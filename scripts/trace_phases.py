"""Per-CTA phase timeline of the pipeline kernels from a -DKB_TRACE build
(scripts/build_variant.sh, selected with KPME_LIB; csrc/trace.h).
usage: KPME_LIB=... python scripts/trace_phases.py cfg3"""
import sys, os, ctypes as C
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2601_18838_b200 import inputs, _lib
from paper_2601_18838_b200.plan import KpmePlan
name = sys.argv[1] if len(sys.argv) > 1 else "cfg3"
w = inputs.workload(name)
plan = KpmePlan(w.cfg, w.grid, w.order, w.dec, w.n)
xyz = torch.as_tensor(w.data.cloud.positions, device='cuda').contiguous()
q = torch.as_tensor(w.data.charges.values, device='cuda').contiguous()
o = torch.empty(w.n, dtype=torch.float64, device='cuda')
flush = torch.empty(256 << 17, dtype=torch.float64, device='cuda')
for _ in range(3):
    flush.zero_()
    plan.execute(xyz, q, o, defer_checks=True)
torch.cuda.synchronize()
lib = C.CDLL(_lib.LIB_PATH)
KERNELS = [("sort2", 0, "tile_keys: 0 start 1 keys 2 ballots 3 bases 4 placed 5 written"),
           ("sort2", 1, "z_tiles_ko: 0 start 1 toff+scan 2 pairs staged 3 counted 4 scanned 5 ranked 6 written"),
           ("interp", 0, "spread: 0 start 1 prologue 2 main loop 3 epilogue"),
           ("interp", 1, "gather: 0 start 1 y/x expansion 2 psi batch 3 particles")]
for unit, k, desc in KERNELS:
    fn = getattr(lib, f"kpme_debug_trace_{unit}", None)
    if fn is None:
        continue
    buf = np.zeros((4096, 10), dtype=np.uint64)
    assert fn(k, buf.ctypes.data_as(C.c_void_p)) == 0
    t = buf[buf[:, 0] > 0].astype(np.int64)
    if os.environ.get("TRACE_SAVE"):
        np.save(f"{os.environ['TRACE_SAVE']}_{unit}{k}.npy", t)
    if not len(t):
        continue
    t0 = t[:, 0].min()
    print(f"{desc}; {len(t)} CTAs")
    prev = 0
    for j in range(1, 7):
        if not (t[:, j] > 10**12).all():
            continue
        d = (t[:, j] - t[:, prev]) / 1e3
        at = (t[:, j] - t0) / 1e3
        print(f"  {prev}->{j}: mean {d.mean():6.2f} min {d.min():6.2f} max {d.max():6.2f} us; mark {j} at {at.min():5.1f}..{at.max():5.1f} (mean {at.mean():5.1f})")
        prev = j
    st = (t[:, 0] - t0) / 1e3
    if os.environ.get("TRACE_DUMP"):
        print("  raw slots 4..6 of the first CTAs:", t[:3, 4:7].tolist())
    if unit == "interp" and k == 0 and (t[:, 6] > 0).all() and (t[:, 6] < 10**9).all():
        print("  spread warp 0 cycles: record issue + wait %.0f (issue alone %.0f), staging %.0f, k-steps %.0f, per-cell drain + contraction %.0f" % (
            t[:, 4].mean(), t[:, 8].mean(), t[:, 5].mean(), t[:, 6].mean(), t[:, 7].mean()))
    if unit == "interp" and k == 1 and (t[:, 7] > 10**12).all():
        print("  gather prologue: tables loaded at %.2f us (CTA-relative mean); warp 0 cycles inside the Horner loops: mean %.0f" % (
            ((t[:, 7] - t[:, 0]) / 1e3).mean(), t[:, 8].mean()))
    if unit == "interp" and k == 1 and (t[:, 5] > 0).all() and (t[:, 5] < 10**9).all():
        # cell-chunk gather, warp 0: cycles waiting for records / evaluating, Horner rounds
        print("  warp 0: wait cycles mean %.0f, work cycles mean %.0f, rounds mean %.1f -> %.0f cycles per round" % (
            t[:, 4].mean(), t[:, 5].mean(), t[:, 6].mean(), t[:, 5].mean() / t[:, 6].mean()))
    last = max(j for j in range(1, 7) if (t[:, j] > 10**12).all())
    life = (t[:, last] - t[:, 0]) / 1e3
    print("  CTA lifetime percentiles 0/10/50/90/100:", np.round(np.percentile(life, [0, 10, 50, 90, 100]), 1))
    sm = t[:, 9]
    per_sm = np.bincount(sm.astype(np.int64))
    print("  CTAs per SM histogram:", dict(zip(*np.unique(per_sm[per_sm > 0], return_counts=True))))
    if os.environ.get("TRACE_DUMP"):
        order = np.argsort(life)
        for c in list(order[:5]) + list(order[-8:]):
            print(f"    cta {c} sm {sm[c]} n_on_sm {per_sm[sm[c]]} marks", np.round((t[c, :8] - t0) / 1e3, 1))
    print(f"  CTA starts {st.min():.1f}..{st.max():.1f} us (mean {st.mean():.1f})")
