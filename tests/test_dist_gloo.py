"""N > 1 host logic on CPU with gloo, world_size 2.

Each rank takes its round-robin share of replay scenarios (shard_round_robin
over seed groups, as bench.py does), replays it, and the per-bucket int64
counters are summed with one all_reduce (gloo here, NCCL on the GPUs).  The
total must equal the unsharded replay bit for bit, and the score/pick block
partition must cover every queue exactly once.  The per-rank replay here is the
oracle (CPU); on the GPU the same plumbing wraps orloj_replay_trace.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import gen
import oracle
from paper_2209_00159_b200 import parallel

NB = len(gen.BUCKET_SLO_MULTS)
SEEDS = 3
N_ARR = 600


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _replay_counters(fam, local_ids):
    tf = gen.c5_trace_family(fam)
    gids, bucket, slo = gen.c5_scenarios(tf, SEEDS)
    gids, bucket, slo = gids[local_ids], bucket[local_ids], slo[local_ids]
    arr, dist_, tb = gen.trace_host(tf, gids, N_ARR)
    off = np.arange(len(gids) + 1, dtype=np.int64) * N_ARR
    r = oracle.replay(oracle.cdf(tf.fam.counts), tf.profile.a, tf.profile.w, off, arr, dist_, tb, slo, nthreads=1)
    return oracle.bucket_counters(r["counters"], bucket, NB)


def _worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        totals = {}
        for fam in gen.C5_FAMILIES:
            u = np.arange(NB * SEEDS)
            mine = parallel.shard_round_robin(u // NB, rank, world)
            t = torch.from_numpy(_replay_counters(fam, mine))
            parallel.allreduce_counters(t)
            totals[fam] = t.numpy()
        lo, hi = parallel.shard_blocks(1000, rank, world)
        cover = torch.zeros(1000, dtype=torch.int64)
        cover[lo:hi] += 1
        dist.all_reduce(cover)
        if rank == 0:
            np.savez(out, cover=cover.numpy(), **totals)
    finally:
        dist.destroy_process_group()


def test_sharded_replay_equals_unsharded(tmp_path):
    out = str(tmp_path / "r.npz")
    mp.spawn(_worker, args=(2, _free_port(), out), nprocs=2, join=True)
    got = np.load(out)
    assert (got["cover"] == 1).all()
    for fam in gen.C5_FAMILIES:
        full = _replay_counters(fam, np.arange(NB * SEEDS))
        assert (got[fam] == full).all(), fam
        assert (full[:, 1] + full[:, 2] + full[:, 3] == full[:, 0]).all()


@pytest.mark.parametrize("world", [1, 2, 3, 8])
def test_partitions(world):
    n = 8192
    seen = np.zeros(n, int)
    for r in range(world):
        lo, hi = parallel.shard_blocks(n, r, world)
        seen[lo:hi] += 1
    assert (seen == 1).all()
    u = np.arange(NB * 256)
    parts = [parallel.shard_round_robin(u // NB, r, world) for r in range(world)]
    assert sorted(np.concatenate(parts).tolist()) == u.tolist()
    for p in parts:                                    # every rank gets every bucket
        assert set((u[p] % NB).tolist()) == set(range(NB)) or world > 256
