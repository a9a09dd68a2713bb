"""Golden replay-policy cases (tests/golden/policy_replay.json) as arrays."""
import json
import os

import numpy as np


def load():
    with open(os.path.join(os.path.dirname(__file__), "golden", "policy_replay.json")) as f:
        return json.load(f)["cases"]


def arrays(case):
    B = case["B"]
    if "counts" in case:
        counts = np.array(case["counts"], np.uint32)
    else:
        counts = np.zeros((len(case["counts_sparse"]), B), np.uint32)
        for d, entries in enumerate(case["counts_sparse"]):
            for i, c in entries:
                counts[d, i] = c
    n = len(case["arrival"])
    # one scenario per request set: a single scenario, constant SLO -> use per-request SLO only if equal
    return dict(counts=counts, a=np.array(case["a"], np.int64), w=np.array(case["w"], np.int64),
                off=np.array([0, n], np.int64), arrival=np.array(case["arrival"], np.int64),
                dist=np.array(case["dist"], np.int32), tb=np.array(case["true_bin"], np.int16),
                slo=np.array(case["slo"], np.int64))
