"""N > 1 replay path with the CUDA kernels.

Two processes share cuda:0 and form a gloo process group (the only GPU this
build gets; on a multi-GPU box bench.py runs the same code with one process per
GPU and NCCL).  Each rank takes its round-robin share of the replay scenarios
(parallel.shard_round_robin over seed groups, exactly as bench.py does), runs
the CUDA replay on it (plain and segmented kernels), and the per-bucket int64
counters are summed with one all_reduce.  The totals must equal the unsharded
CUDA replay of all scenarios bit for bit, for every family, and the oracle in
follow mode must agree with the unsharded run on every scenario.
"""
import os
import socket

import numpy as np
import pytest

import gen
import oracle
import _parity as par

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a GPU", allow_module_level=True)

import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402

NB = len(gen.BUCKET_SLO_MULTS)
SEEDS = 6          # 48 scenarios per family
N_ARR = 12_000
SEGMENTS = 4


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _family_counters(fam, local_ids, segments):
    import paper_2209_00159_b200 as orj
    import workloads as wl
    f = wl.C5Family(fam, local_ids=local_ids, n_arr=N_ARR, seeds_per_bucket=SEEDS)
    tab, _ = orj.replay_trace(f.store, f.profile, f.trace, segments=segments)
    torch.cuda.synchronize()
    return tab.cpu()


def _worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2209_00159_b200 import parallel
    try:
        res = {}
        u = np.arange(NB * SEEDS)
        mine = parallel.shard_round_robin(u // NB, rank, world)
        for fam in gen.C5_FAMILIES:
            for g in (1, SEGMENTS):
                t = _family_counters(fam, mine, g)
                parallel.allreduce_counters(t)          # gloo on CPU tensors (NCCL on the GPUs in bench.py)
                res[f"{fam}/{g}"] = t.numpy()
                res[f"{fam}/{g}/rate"] = parallel.finish_rate(t).numpy()
        if rank == 0:
            np.savez(out, **res)
    finally:
        dist.destroy_process_group()


def test_cuda_shards_allreduce_equal_unsharded(tmp_path):
    out = str(tmp_path / "r.npz")
    ctx = mp.get_context("spawn")
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, out)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=600)
        assert p.exitcode == 0, f"rank exited with {p.exitcode}"
    got = np.load(out)
    import paper_2209_00159_b200 as orj
    import workloads as wl
    for fam in gen.C5_FAMILIES:
        full = _family_counters(fam, None, 1).numpy()
        assert (full[:, 1] + full[:, 2] + full[:, 3] == full[:, 0]).all()
        assert full[:, 0].sum() == NB * SEEDS * N_ARR
        for g in (1, SEGMENTS):
            assert (got[f"{fam}/{g}"] == full).all(), (fam, g)
            assert np.array_equal(got[f"{fam}/{g}/rate"], full[:, 1] / np.maximum(full[:, 0], 1))
        # the unsharded CUDA run itself: oracle in follow mode, counters bit-exact per scenario
        f = wl.C5Family(fam, n_arr=N_ARR, seeds_per_bucket=SEEDS)
        S = f.num_scenarios
        per_scen = orj.Trace(f.trace.offsets, f.trace.arrival, f.trace.dist, f.trace.true_bin, f.trace.slo,
                             torch.arange(S, dtype=torch.int32, device="cuda"), S)
        pb, log = orj.replay_trace(f.store, f.profile, per_scen, decision_log=True)
        torch.cuda.synchronize()
        ref = oracle.replay(oracle.cdf(f.tf.fam.counts), f.tf.profile.a, f.tf.profile.w, f.offsets_np,
                            f.trace.arrival.cpu().numpy(), f.trace.dist.cpu().numpy(),
                            f.trace.true_bin.cpu().numpy(), f.slo_np, follow_log=log.cpu().numpy())
        par.check_replay_follow(ref, pb.cpu().numpy(), f"dist-shared/{fam}")
