"""Profiling driver: each C2 scoring-model variant of bench.run_model_variants
launched twice (warm-up + the profiled launch), eagerly, in the bench's order,
for an ncu launch list (no timing is reported from here)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import gen  # noqa: E402
import paper_2209_00159_b200 as orj  # noqa: E402
import workloads as wl  # noqa: E402


def main():
    dev = torch.device("cuda", 0)
    cfg = gen.config2()
    store = wl.score_store(cfg, dev)
    qs = wl.device_queues(cfg.queues, dev, with_arrival=False)
    prof = wl.profile(cfg.profile)
    for name, tab, interp, st in bench.model_variant_specs(cfg, prof):
        model = orj.ScoreModel(tab, interpolate=interp, steps=st, device=dev)
        for _ in range(2):
            model.score(store, qs)
        torch.cuda.synchronize()


if __name__ == "__main__":
    main()
