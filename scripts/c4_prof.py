"""Profiling driver: C4 (1,048,576 static-CNN queues x 32) and C2 picks, a few
launches each (for ncu; no timing is reported from here)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import gen  # noqa: E402
import paper_2209_00159_b200 as orj  # noqa: E402
import workloads as wl  # noqa: E402


def main():
    which = sys.argv[1] if len(sys.argv) > 1 else "C4"
    cfg = gen.config4() if which == "C4" else gen.config2()
    store = wl.score_store(cfg)
    prof = wl.profile(cfg.profile)
    qs = wl.device_queues(cfg.queues, with_arrival=False)
    Q = cfg.queues.Q
    bk = torch.empty(Q, dtype=torch.int32, device="cuda")
    bE = torch.empty(Q, dtype=torch.float32, device="cuda")
    for _ in range(int(sys.argv[2]) if len(sys.argv) > 2 else 4):
        orj.pick_batch(store, prof, qs, bk, bE)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20):
        orj.pick_batch(store, prof, qs, bk, bE)
    e1.record()
    torch.cuda.synchronize()
    print(f"{which}: {e0.elapsed_time(e1) / 20 * 1e3:.1f} us per pick")


if __name__ == "__main__":
    main()
