"""Parity helpers for the GPU tests (test infrastructure: may use the oracle)."""
import numpy as np

import oracle

P_TOL = 1e-5          # north star: probabilities within 1e-5 absolute


def e_tol(kmax):
    """E_k within 1e-5 * k (SURVEY §8(c) tolerances; derivation DESIGN.md §5)."""
    return 1e-5 * np.arange(1, kmax + 1)


def oracle_score(counts, prof_a, prof_w, q, want_P=False, want_EL=False):
    return oracle.score(oracle.cdf(counts), prof_a, prof_w, q.offsets, q.deadline, q.dist, q.now,
                        want_P=want_P, want_EL=want_EL)


def check_E(E_gpu, E_or, lens, kmax):
    """Element-wise E parity; entries k > K_q must be exactly 0."""
    K = np.minimum(lens, kmax)
    err = np.abs(E_gpu.astype(np.float64) - E_or)
    assert (err <= e_tol(kmax)[None, :] + 1e-7).all(), f"max E err {err.max()}"
    mask = np.arange(1, kmax + 1)[None, :] > K[:, None]
    assert (E_gpu[mask] == 0).all()
    return err.max()


def check_pick(bk_gpu, bE_gpu, E_gpu, E_or, bk_or, lens, kmax):
    """k* bit-exact except documented ties: k_g != k_o is accepted iff
    E_or[k_o] - E_or[k_g] <= |E_gpu[k_g] - E_or[k_g]| + |E_gpu[k_o] - E_or[k_o]|,
    each error within 1e-5 k.  Returns the number of ties."""
    K = np.minimum(lens, kmax)
    assert ((bk_gpu == 0) == (K == 0)).all()
    ties = 0
    for q in np.nonzero(bk_gpu != bk_or)[0]:
        kg, ko = int(bk_gpu[q]), int(bk_or[q])
        eg = abs(float(E_gpu[q, kg - 1]) - E_or[q, kg - 1])
        eo = abs(float(E_gpu[q, ko - 1]) - E_or[q, ko - 1])
        assert eg <= 1e-5 * kg + 1e-7 and eo <= 1e-5 * ko + 1e-7
        assert E_or[q, ko - 1] - E_or[q, kg - 1] <= eg + eo + 1e-12, f"queue {q}: k_gpu={kg} k_oracle={ko}"
        ties += 1
    nz = K > 0
    # best_E is E_gpu[k*] (pick and score variants evaluate the same arithmetic)
    idx = np.nonzero(nz)[0]
    assert (bE_gpu[idx] == E_gpu[idx, bk_gpu[idx] - 1]).all()
    assert (bE_gpu[~nz] == 0).all()
    return ties


def check_P(P_gpu, P_or, lens, kmax):
    K = np.minimum(lens, kmax)
    tri = np.concatenate([np.full(k, k) for k in range(1, kmax + 1)])  # k of each packed entry
    valid = tri[None, :] <= K[:, None]
    err = np.abs(P_gpu.astype(np.float64) - P_or)[valid]
    assert err.size == 0 or err.max() <= P_TOL, f"max P err {err.max()}"
    assert (P_gpu[valid] >= 0).all() and (P_gpu[valid] <= 1).all()
    return 0.0 if err.size == 0 else err.max()


def record(kind: str, **stats):
    """Append a parity statistic (e.g. tie counts) as one JSON line to the file
    named by $ORLOJ_PARITY_LOG (evidence for DESIGN.md); no-op otherwise."""
    import json
    import os
    path = os.environ.get("ORLOJ_PARITY_LOG")
    if path:
        with open(path, "a") as f:
            f.write(json.dumps({"kind": kind, **{k: (v.item() if hasattr(v, "item") else v)
                                                 for k, v in stats.items()}}) + "\n")


def check_replay_follow(ref, counters_gpu, label: str, tie_rate: float = 1e-5, free=None, log_gpu=None):
    """Replay parity in follow mode: every GPU decision lies in
    the oracle's tie set, the integer counters are bit-exact, and the number of
    GPU choices that differ from the oracle's own choice (documented ties) is
    reported and bounded by `tie_rate` x decisions (+1 for a lone tie in a
    tiny case).  With the oracle's free run `free`, every scenario without a
    differing decision must equal it bit for bit (counters, and the log when
    both logs are given): the free run can only diverge after a tie."""
    ties = ref["ties"]
    bad = np.nonzero(ties[:, 2] != -1)[0]
    assert bad.size == 0, f"{label}: scenario {bad[:5]} has a GPU decision outside the oracle tie set"
    assert (ref["counters"] == counters_gpu).all(), f"{label}: counters differ in follow mode"
    dec, diff = int(ties[:, 0].sum()), int(ties[:, 1].sum())
    clean = ties[:, 1] == 0
    out = {"decisions": dec, "differing_choices": diff, "scenarios": len(ties),
           "scenarios_with_ties": int((~clean).sum())}
    if free is not None:
        same = (free["counters"] == counters_gpu).all(1)
        assert same[clean].all(), f"{label}: a tie-free scenario differs from the oracle's free run"
        out["free_run_identical_scenarios"] = int(same.sum())
        if log_gpu is not None and free.get("log") is not None and clean.all():
            assert (free["log"] == log_gpu).all(), f"{label}: free-run log differs"
    record("replay_ties", label=label, **out)
    assert diff <= tie_rate * dec + 1, f"{label}: {diff} differing choices in {dec} decisions"
    return out
