#!/usr/bin/env python
"""bench.py — scheduling decisions/s of the B200 Orloj batch-scoring path.

Default (N = 1): workload C3: 65,536 queues x 256 requests with
per-request 256-bin histograms (16.8 M rows, 17.2 GB log2-CDF store in HBM),
kmax = 256.  One step = one orloj_pick_batch over all queues (rows a1-a6 of
SURVEY §8(a)); inputs (17.4 GB per step) are larger than L2, so no flush is
needed between steps.  The store is built once, off the timed region (a0; the
paper's profiler is off the critical path).

Also measured in the same run (sub-objects of the one JSON line):
  e2e          the same pick through orloj_pick_batch_host, with the queue
               arrays copied from pinned host memory and results copied back
               inside the timed region;
  replay       the C5 trace-replay sweep (rows a7-a8): 4 families x 8 SLO
               buckets x 256 seeds x 100k arrivals, scenarios sharded
               round-robin over ranks, one NCCL all-reduce of the counters;
  roofline     HBM roofline of the dominant kernel (the pick kernel);
  cpu_baseline the fp64 oracle on a bounded C3 sample on the host cores.

Multi-GPU (torchrun): every rank picks its own C3 instance (weak scaling, no
collective on the score path); value = all ranks' decisions / max-over-ranks
time.  --impl reference times the oracle (the tier's reference arm).
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "scheduling decisions/sec and candidate batches/sec @1/2/4/8 B200; HBM GB/s % peak"
WORKLOAD = ("C3: 65,536 queues x 256 requests x 256-bin per-request histograms (BART-CNN-like, "
            "mean 774.66 / P99 1101.99 ms), kmax = 256, 16.8 M permuted 1 KB rows (17.2 GB store)")


def nvtx(name):
    """NVTX range around a bench leg (nsys attribution; a no-op without a tool)."""
    import torch
    return torch.cuda.nvtx.range(name)


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="orloj", choices=["orloj", "reference"])
    ap.add_argument("--queues", type=int, default=65536)
    ap.add_argument("--kmax", type=int, default=256)
    ap.add_argument("--no-replay", action="store_true")
    ap.add_argument("--replay-seeds", type=int, default=256, help="seeds per (family, bucket)")
    ap.add_argument("--replay-arrivals", type=int, default=100_000)
    ap.add_argument("--replay-reps", type=int, default=2)
    ap.add_argument("--replay-segments", default="auto,last=auto",
                    help="segments per scenario of the segmented replay ('auto' or an int; 1 = plain kernel; "
                         "'fam=G' per family; 'last=G' / 'last=xM' / 'last=auto' for the family launched last)")
    ap.add_argument("--seg-sweep-n", default="1,2,4,8")
    ap.add_argument("--seg-sweep-g", default="1,2,4,8,16,32,64,auto")
    ap.add_argument("--replay-seg-sweep", action="store_true",
                    help="diagnostic: time the C5 sweep and its rank-0 shards for several segment counts")
    ap.add_argument("--scenario-order", default="seed", choices=["seed", "bucket"],
                    help="order of a rank's C5 scenarios in its trace (seed groups, or SLO bucket by bucket)")
    ap.add_argument("--no-shard-proxy", action="store_true")
    ap.add_argument("--proxy-segments", default=None, help="segments per scenario in the shard proxy (default: as --replay-segments)")
    ap.add_argument("--no-policies", action="store_true", help="skip the replay policy-variant sweep")
    ap.add_argument("--policy-seeds", type=int, default=32)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--e2e-chunks", type=int, default=12)
    ap.add_argument("--e2e-streams", type=int, default=2)
    ap.add_argument("--no-extra", action="store_true", help="skip the C2 / C4 workload lines")
    ap.add_argument("--cpu-seconds", type=float, default=12.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--ncu", action="store_true", help="profiling mode: only the timed pick loop")
    ap.add_argument("--only-replay", action="store_true", help="profiling mode: only the replay sweep")
    return ap.parse_args()


def dist_env():
    return int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)), int(os.environ.get("LOCAL_RANK", 0))


def free_port() -> int:
    import socket
    with socket.socket(socket.AF_INET, socket.SOCK_STREAM) as so:
        so.bind(("127.0.0.1", 0))
        return so.getsockname()[1]


def self_launch(args) -> int:
    """`--gpus N > 1` outside torchrun: re-run this command as N ranks under
    torch.distributed.run (one process per GPU, rendezvous on 127.0.0.1), the
    launch the driver uses.  N must not exceed the visible GPUs unless
    ORLOJ_BENCH_SHARE_GPU=1 (functional check: every rank on cuda:0, gloo)."""
    import subprocess
    import torch
    have = torch.cuda.device_count()
    if args.gpus > have and os.environ.get("ORLOJ_BENCH_SHARE_GPU") != "1":
        print(json.dumps({"error": f"--gpus {args.gpus} but only {have} GPU(s) visible",
                          "hint": "run on a box with enough GPUs (or ORLOJ_BENCH_SHARE_GPU=1 for a functional "
                                  "check with every rank on cuda:0)"}), flush=True)
        return 2
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr=127.0.0.1", f"--master-port={free_port()}", os.path.abspath(__file__), *sys.argv[1:]]
    return subprocess.call(cmd)


# ----------------------------------------------------------------------------
# clocks sampled during the timed region (NVML)
# ----------------------------------------------------------------------------

class ClockSampler:
    REASONS = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap",
               0x8: "hw_slowdown", 0x10: "sync_boost", 0x20: "sw_thermal_slowdown",
               0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting"}

    def __init__(self, index: int, period_s: float = 0.01):
        self.samples, self.reasons = [], set()
        self.period = period_s
        self._stop = threading.Event()
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception as e:  # pragma: no cover
            self.nv, self.err = None, str(e)

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                r = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for bit, name in self.REASONS.items():
                    if r & bit and name != "gpu_idle":
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(self.period)

    def __enter__(self):
        if self.nv:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        if self.nv:
            self._stop.set()
            self.t.join()

    def summary(self):
        if not self.nv:
            return {"error": getattr(self, "err", "nvml unavailable")}
        return {"sm_mhz": float(np.median(self.samples)) if self.samples else None,
                "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons), "samples": len(self.samples)}


def measured_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, STREAM-style copy)"
    return 6650.0, "fallback (B200_PROFILING.md: 6.65 TB/s)"


def ncu_traffic():
    """dram bytes per launch of the pick kernel from the committed ncu --set full summary."""
    p = os.path.join(ROOT, "profiles", "ncu_c3_pick_summary.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return d.get("dram_bytes_per_launch")
    return None


# ----------------------------------------------------------------------------
# oracle timing (cpu_baseline leg and the --impl reference arm)
# ----------------------------------------------------------------------------

def oracle_c3_sample(cfg, nq: int, start: int = 0):
    import gen
    sub = cfg.queues.subset(np.arange(start, start + nq))
    rows = gen.rows_host(cfg.row_seed, sub.dist.astype(np.uint64), cfg.fam.counts)
    local = gen.Queues(sub.offsets, sub.arrival, sub.deadline, np.arange(len(sub.dist), dtype=np.int32), sub.now)
    return rows, local


def time_oracle_c3(cfg, seconds: float, chunk: int = 64, keep=None):
    """Run the oracle on consecutive chunks of C3 queues until `seconds` of work.
    keep: a list that receives (start, oracle result) per chunk (untimed use:
    the bench's parity summary compares them with the GPU's k*)."""
    import oracle
    done, t_or, start = 0, 0.0, 0
    while t_or < seconds and start + chunk <= cfg.queues.Q:
        rows, local = oracle_c3_sample(cfg, chunk, start)
        t0 = time.perf_counter()
        F = oracle.cdf(rows)
        res = oracle.score(F, cfg.profile.a, cfg.profile.w, local.offsets, local.deadline, local.dist, local.now)
        t_or += time.perf_counter() - t0
        if keep is not None:
            keep.append((start, res))
        done += chunk
        start += chunk
    return done, t_or, oracle.max_threads()


def c3_parity_summary(kept, bk_gpu, kmax):
    """k* of the GPU's timed C3 pick against the oracle on the cpu_baseline
    sample: equal, or a difference within the E tolerance (a documented tie:
    E_or[k_o] - E_or[k_g] <= 1e-5 (k_o + k_g)), else a mismatch."""
    eq = tie = bad = 0
    for start, res in kept:
        ko = np.asarray(res["best_k"])
        E = np.asarray(res["E"])
        kg = bk_gpu[start:start + len(ko)]
        for j in np.nonzero(kg != ko)[0]:
            a, g = int(ko[j]), int(kg[j])
            if g >= 1 and E[j, a - 1] - E[j, g - 1] <= 1e-5 * (a + g):
                tie += 1
            else:
                bad += 1
        eq += int((kg == ko).sum())
    return {"queues": eq + tie + bad, "k_equal": eq, "k_documented_ties": tie, "k_mismatches": bad,
            "source": "the cpu_baseline leg's fp64 oracle output on the same queues vs the timed GPU pick"}


def time_oracle_configs(replay_scenarios: int = 256):
    """The oracle on the other §8(d) configs, on all host cores (SURVEY §8(d)
    "Oracle timing"): C1 brute force + O1, C2 and C4 in full, and a C5 subset
    spanning every family and bucket (O2, free mode)."""
    import gen
    import oracle
    out = {"host_threads": oracle.max_threads(), "nproc": os.cpu_count()}
    try:
        with open("/proc/cpuinfo") as f:
            out["cpu_model"] = next((l.split(":", 1)[1].strip() for l in f if l.startswith("model name")), None)
    except OSError:
        pass
    c = gen.config1()
    q = c.queues
    t0 = time.perf_counter()
    oracle.bruteforce(c.fam.counts, c.profile.a, c.profile.w, q.deadline, q.dist, int(q.now[0]))
    t1 = time.perf_counter()
    oracle.score(oracle.cdf(c.fam.counts), c.profile.a, c.profile.w, q.offsets, q.deadline, q.dist, q.now)
    t2 = time.perf_counter()
    out["C1"] = {"bruteforce_ms": 1e3 * (t1 - t0), "o1_ms": 1e3 * (t2 - t1)}
    for name, cfg in (("C2", gen.config2()), ("C4", gen.config4())):
        q = cfg.queues
        F = oracle.cdf(cfg.fam.counts)
        t0 = time.perf_counter()
        oracle.score(F, cfg.profile.a, cfg.profile.w, q.offsets, q.deadline, q.dist, q.now)
        dt = time.perf_counter() - t0
        out[name] = {"queues": q.Q, "seconds": dt, "decisions_per_s": q.Q / dt}
    nb = len(gen.BUCKET_SLO_MULTS)
    per = max(1, replay_scenarios // (len(gen.C5_FAMILIES) * nb))
    dec, secs, arrivals = 0, 0.0, 0
    for fam in gen.C5_FAMILIES:
        tf = gen.c5_trace_family(fam)
        gids, bucket, slo = gen.c5_scenarios(tf, per)
        arr, dist, tb = gen.trace_host(tf, gids, gen.C5_ARRIVALS)
        off = np.arange(len(gids) + 1, dtype=np.int64) * gen.C5_ARRIVALS
        t0 = time.perf_counter()
        r = oracle.replay(oracle.cdf(tf.fam.counts), tf.profile.a, tf.profile.w, off, arr, dist, tb, slo)
        secs += time.perf_counter() - t0
        dec += int(r["ties"][:, 0].sum())
        arrivals += len(arr)
    out["C5"] = {"scenarios": per * len(gen.C5_FAMILIES) * nb, "arrivals": arrivals, "decisions": dec,
                 "seconds": secs, "decisions_per_s": dec / secs}
    return out


def run_reference(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return
    import gen
    cfg = gen.config3(Q=args.queues, kmax=args.kmax)
    per_step = 128
    import oracle
    secs = []
    for s in range(args.warmup + args.steps):
        rows, local = oracle_c3_sample(cfg, per_step, (s * per_step) % (cfg.queues.Q - per_step))
        t0 = time.perf_counter()
        oracle.score(oracle.cdf(rows), cfg.profile.a, cfg.profile.w, local.offsets, local.deadline, local.dist,
                     local.now)
        if s >= args.warmup:
            secs.append(time.perf_counter() - t0)
    t = float(np.sum(secs))
    val = per_step * len(secs) / t
    cores = oracle.max_threads()
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": val, "unit": "decisions/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1000 * t / len(secs), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": WORKLOAD, "step": f"{per_step} C3 queues on the host (bounded sample)"},
        "cpu_baseline": {"value": val, "unit": "decisions/s", "cores": cores, "kind": "oracle",
                         "sample": f"{per_step} consecutive C3 queues per step, fp64 oracle, all host threads"},
        "e2e": {"value": val, "unit": "decisions/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }), flush=True)


# ----------------------------------------------------------------------------
# GPU arm
# ----------------------------------------------------------------------------

def main():
    args = parse()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(self_launch(args))
    if args.impl == "reference":
        return run_reference(args)
    import torch
    import torch.distributed as dist

    import gen
    import paper_2209_00159_b200 as orj
    import workloads as wl

    rank, world, local = dist_env()
    # ORLOJ_BENCH_SHARE_GPU=1: every rank on cuda:0 with gloo collectives -- a
    # functional check of the N > 1 path on a one-GPU box (its timings mean nothing)
    shared = os.environ.get("ORLOJ_BENCH_SHARE_GPU") == "1"
    if shared:
        local = 0
    torch.cuda.set_device(local)
    if world > 1:
        if shared:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.device("cuda", local)
    comm = None
    if world > 1:
        comm = {"backend": dist.get_backend(), "world_size": world, "local_rank_device": local,
                "nccl_version": ".".join(map(str, torch.cuda.nccl.version())) if not shared else None,
                "shared_gpu_functional_check": shared}

    def barrier():
        if world > 1:
            dist.barrier()

    def max_over_ranks(x: float) -> float:
        if world == 1:
            return x
        tt = torch.tensor([x], dtype=torch.float64, device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        return float(tt.item())

    if args.replay_seg_sweep:
        out = {}
        for N in [int(x) for x in args.seg_sweep_n.split(",")]:
            sf = build_replay(args, 0, N, dev)
            for G in args.seg_sweep_g.split(","):
                ms, tabs, _ = time_replay(sf, args.replay_reps, dev, lambda: None, lambda x: x, reduce=False,
                                          segments=G)
                out[f"N{N}/G{G}"] = {"ms": round(ms, 3), "segments": list(time_replay.segments),
                                     "decisions": int(tabs[:, :, 4].sum()), "stitch": time_replay.stats}
                print(json.dumps({f"N{N}/G{G}": out[f"N{N}/G{G}"]}), flush=True)
            del sf
        print(json.dumps({"replay_seg_sweep": out}), flush=True)
        return

    if args.only_replay:
        r = run_replay(args, rank, world, dev, barrier, max_over_ranks)
        if rank == 0:
            print(json.dumps({"replay": r}), flush=True)
        return

    # ---------------- C3 pick: setup (untimed) ----------------
    cfg = gen.config3(Q=args.queues, kmax=args.kmax, instance=rank)
    store = wl.c3_store(cfg, dev)
    prof = wl.profile(cfg.profile)
    qn = cfg.queues
    qs = wl.device_queues(qn, dev, with_arrival=False)
    Q = qn.Q
    K = np.minimum(np.diff(qn.offsets), cfg.kmax)
    cands = int(K.sum())
    B = cfg.fam.B
    algo_bytes = (cands * B * 4                      # log2-CDF rows gathered
                  + int(K.sum()) * (8 + 4)           # deadline + dist id per candidate member
                  + (Q + 1) * 8 + Q * 8              # offsets, now
                  + Q * (4 + 4))                     # best_k, best_E
    bk = torch.empty(Q, dtype=torch.int32, device=dev)
    bE = torch.empty(Q, dtype=torch.float32, device=dev)
    stream = torch.cuda.current_stream()
    for _ in range(args.warmup):
        orj.pick_batch(store, prof, qs, bk, bE, stream)
    torch.cuda.synchronize()
    barrier()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        torch.cuda.synchronize()
        ev0.record(stream)
        for _ in range(args.steps):
            orj.pick_batch(store, prof, qs, bk, bE, stream)
        ev1.record(stream)
        torch.cuda.synchronize()
    barrier()
    ms_total = ev0.elapsed_time(ev1)
    ms_total = max_over_ranks(ms_total)
    ms_step = ms_total / args.steps
    value = world * Q / (ms_step / 1e3)
    cand_s = world * cands / (ms_step / 1e3)
    achieved = algo_bytes / (ms_step / 1e3) / 1e9
    peak, peak_src = measured_peaks()
    traffic = ncu_traffic()
    result = {
        "metric": METRIC, "value": value, "unit": "decisions/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f32", "data": "synthetic (seeded; SURVEY §8(d) recipe, DESIGN.md §4)",
        "config": {"workload": WORKLOAD, "queues_per_gpu": Q, "requests_per_queue": int(np.diff(qn.offsets)[0]),
                   "bins": B, "kmax": cfg.kmax, "global_queues": world * Q,
                   "l2": "inputs larger than L2 (17.4 GB read per step); no flush",
                   "parallelism": f"queues sharded, {world} independent C3 instances, no collective",
                   "seed": gen.SEED_BASE + 3},
        "candidates_per_s": cand_s,
        "hbm_gbs_algorithmic": achieved,
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                     "traffic": traffic, "kernel": "score_kernel<8,8,PICK,STREAM> (orloj_pick_batch)",
                     "algorithmic_bytes_per_launch": algo_bytes, "peak_source": peak_src,
                     "note": "the peak is a read+write copy; this kernel's bytes are >99.9 % reads (a read-only "
                             "stream can run a little above the copy figure); traffic = ncu DRAM bytes per launch"},
        "gpu_launches": args.steps,
        "clocks": clk.summary(),
    }
    if comm:
        result["comm"] = comm
    if args.ncu:
        if rank == 0:
            print(json.dumps(result), flush=True)
        return

    # ---------------- C3 secondary shapes: K = 64, identity row layout ----------------
    if not args.no_extra:
        var = {}
        kk = min(64, cfg.kmax)
        p64 = orj.LatencyProfile(cfg.profile.a[:kk], cfg.profile.w[:kk])
        ident = orj.Queues(qs.offsets, qs.deadline, torch.arange(qn.N, dtype=torch.int32, device=dev), qs.now)
        for vname, pr_, qq, kq in (("C3_k64", p64, qs, kk), ("C3_identity_rows", prof, ident, cfg.kmax)):
            for _ in range(2):
                orj.pick_batch(store, pr_, qq, bk, bE, stream)
            v0, v1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            v0.record(stream)
            for _ in range(10):
                orj.pick_batch(store, pr_, qq, bk, bE, stream)
            v1.record(stream)
            torch.cuda.synchronize()
            vms = max_over_ranks(v0.elapsed_time(v1)) / 10
            vc = int(np.minimum(np.diff(qn.offsets), kq).sum())
            vb = vc * B * 4 + vc * 12 + (Q + 1) * 8 + Q * 16
            var[vname] = {"kmax": kq, "ms_per_pick": vms, "decisions_per_s": world * Q / (vms / 1e3),
                          "candidates_per_s": world * vc / (vms / 1e3),
                          "hbm_frac_algorithmic": vb / (vms / 1e3) / 1e9 / peak}
        var["C3_identity_rows"]["note"] = "dist_id = identity (each queue's rows contiguous) instead of the permutation"
        result["c3_variants"] = var
        del ident

    # ---------------- e2e: host buffers through orloj_pick_batch_host ----------------
    if not args.no_e2e:
        pin = lambda a, dt: torch.from_numpy(np.ascontiguousarray(a, dtype=dt)).pin_memory()  # noqa: E731
        h_off, h_dl = pin(qn.offsets, np.int64), pin(qn.deadline, np.int64)
        h_dist, h_now = pin(qn.dist, np.int32), pin(qn.now, np.int64)
        hp = orj.HostPicker(store, prof, qn.offsets, chunks=args.e2e_chunks, streams=args.e2e_streams, device=dev)
        for _ in range(max(1, args.warmup)):
            hp.pick(h_off, h_dl, h_dist, h_now, stream)
        torch.cuda.synchronize()
        barrier()
        e_steps = max(5, args.steps // 5)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(e_steps):
            hp.pick(h_off, h_dl, h_dist, h_now, stream)
        e1.record(stream)
        torch.cuda.synchronize()
        barrier()
        e_ms = max_over_ranks(e0.elapsed_time(e1)) / e_steps
        assert (hp.best_k.numpy() == bk.cpu().numpy()).all()
        result["e2e"] = {"value": world * Q / (e_ms / 1e3), "unit": "decisions/s",
                         "h2d_bytes_per_step": hp.h2d_bytes(), "d2h_bytes_per_step": hp.d2h_bytes(),
                         "ms_per_step": e_ms, "steps": e_steps,
                         "path": f"orloj_pick_batch_host: pinned host queues -> H2D -> kernel -> D2H, "
                                 f"{args.e2e_chunks} chunks pipelined on {args.e2e_streams} streams"}
        del hp

    # ---------------- cpu baseline (rank 0, N = 1 only) ----------------
    if world == 1 and not args.no_cpu_baseline:
        kept = []
        n, secs, cores = time_oracle_c3(cfg, args.cpu_seconds, keep=kept)
        result["cpu_baseline"] = {"value": n / secs, "unit": "decisions/s", "cores": cores, "kind": "oracle",
                                  "sample": f"first {n} C3 queues (256 x 256 bins, kmax 256), fp64 oracle, "
                                            f"{secs:.1f} s on {cores} host threads"}
        result["parity"] = c3_parity_summary(kept, bk.cpu().numpy(), cfg.kmax)
        result["oracle_by_config"] = time_oracle_configs()
    else:
        result["cpu_baseline"] = None

    del store, qs
    torch.cuda.empty_cache()

    # ---------------- other workload shapes (C2 SkipNet-like, C4 static CNN) ----------------
    if not args.no_extra:
        with nvtx("workloads"):
            result["workloads"] = run_other_workloads(args, dev, max_over_ranks, world)

    # ---------------- replay sweep (C5) ----------------
    if not args.no_replay:
        with nvtx("replay"):
            result["replay"] = run_replay(args, rank, world, dev, barrier, max_over_ranks)

    if rank == 0:
        print(json.dumps(result), flush=True)
    if world > 1:
        dist.destroy_process_group()


def run_other_workloads(args, dev, max_over_ranks, world):
    """Decisions/s on the other §8(d) score shapes (same kernel family):
    C2 (1,024 SkipNet-like queues x 64, kmax 32, B 64): 100 back-to-back picks
    captured in one CUDA graph; C4 (1,048,576 static-CNN queues x 32, point
    masses, B 32): one pick per step."""
    import torch

    import gen
    import paper_2209_00159_b200 as orj
    import workloads as wl

    out = {}
    stream = torch.cuda.Stream(dev)
    planner_k = None
    c2_best_k = None
    for name, cfg, reps in (("C2", gen.config2(), 100), ("C4", gen.config4(), 1), ("C4-near", gen.config4(near=True), 1)):
        store = wl.score_store(cfg, dev)
        prof = wl.profile(cfg.profile)
        qs = wl.device_queues(cfg.queues, dev, with_arrival=False)
        Q = cfg.queues.Q
        cands = int(np.minimum(np.diff(cfg.queues.offsets), cfg.kmax).sum())
        bk = torch.empty(Q, dtype=torch.int32, device=dev)
        bE = torch.empty(Q, dtype=torch.float32, device=dev)
        with torch.cuda.stream(stream):
            for _ in range(3):
                orj.pick_batch(store, prof, qs, bk, bE, stream)
        torch.cuda.synchronize()
        if reps > 1:
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=stream):
                for _ in range(reps):
                    orj.pick_batch(store, prof, qs, bk, bE, stream)
            run = g.replay
        else:
            def run():
                orj.pick_batch(store, prof, qs, bk, bE, stream)
        with torch.cuda.stream(stream):
            run()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            iters = 20
            e0.record(stream)
            for _ in range(iters):
                run()
            e1.record(stream)
        torch.cuda.synchronize()
        ms = max_over_ranks(e0.elapsed_time(e1)) / (iters * reps)
        out[name] = {"workload": cfg.name, "queues": Q, "kmax": cfg.kmax, "bins": cfg.fam.B,
                     "us_per_pick": 1e3 * ms, "decisions_per_s": world * Q / (ms / 1e3),
                     "candidates_per_s": world * cands / (ms / 1e3),
                     "timing": f"{iters} x " + (f"CUDA graph of {reps} picks" if reps > 1 else "1 pick")}
        if name == "C2":
            c2_best_k = bk.cpu().numpy()
        if name == "C4":
            planner_k = bk.cpu().numpy()  # == the constant-latency planner, bit for bit (tests)
        if name == "C4-near" and planner_k is not None and len(planner_k) == Q:
            out[name]["agreement_with_planner"] = float((bk.cpu().numpy() == planner_k).mean())
        del store, qs
    torch.cuda.empty_cache()
    with nvtx("C2-HBM"):
        out["C2-HBM"] = run_c2_hbm(dev, max_over_ranks, world, c2_best_k)
    with nvtx("C1_latency"):
        out["C1_latency"] = run_c1_latency(dev)
    with nvtx("P1"):
        out["P1"] = run_priority(dev, max_over_ranks, world)
    with nvtx("C2_model_variants"):
        out["C2_model_variants"] = run_model_variants(dev, max_over_ranks, world)
    return out


def run_c2_hbm(dev, max_over_ranks, world, c2_best_k):
    """C2-HBM: the C2 queues with one store row per request
    (65,536 rows, 16.8 MB: the TMA row-ring path instead of the shared-memory
    store), 100 picks per CUDA graph.  Each row equals its request's
    application row, so k* must equal C2's bit for bit."""
    import torch

    import gen
    import paper_2209_00159_b200 as orj
    import workloads as wl

    cfg = gen.config2()
    q = cfg.queues
    N = int(q.offsets[-1])
    counts = np.ascontiguousarray(cfg.fam.counts[q.dist])             # [N][B]: request j's own row
    store = orj.HistogramStore.from_counts(counts, cfg.fam.bin_ticks, dev)
    qs = orj.Queues(wl.t(q.offsets, np.int64, dev), wl.t(q.deadline, np.int64, dev),
                    wl.t(np.arange(N, dtype=np.int32), np.int32, dev), wl.t(q.now, np.int64, dev))
    prof = wl.profile(cfg.profile)
    bk = torch.empty(q.Q, dtype=torch.int32, device=dev)
    bE = torch.empty(q.Q, dtype=torch.float32, device=dev)
    stream = torch.cuda.Stream(dev)
    with torch.cuda.stream(stream):
        for _ in range(3):
            orj.pick_batch(store, prof, qs, bk, bE, stream)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=stream):
        for _ in range(100):
            orj.pick_batch(store, prof, qs, bk, bE, stream)
    with torch.cuda.stream(stream):
        g.replay()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(20):
            g.replay()
        e1.record(stream)
    torch.cuda.synchronize()
    ms = max_over_ranks(e0.elapsed_time(e1)) / 2000
    same = None if c2_best_k is None else bool((bk.cpu().numpy() == c2_best_k).all())
    K = np.minimum(np.diff(q.offsets), cfg.kmax)
    return {"workload": "C2 queues (1,024 x 64, kmax 32, B 64) over 65,536 per-request rows (16.8 MB store)",
            "us_per_pick": 1e3 * ms, "decisions_per_s": world * q.Q / (ms / 1e3),
            "row_bytes_per_pick": int(K.sum()) * cfg.fam.B * 4, "best_k_equals_C2": same,
            "timing": "20 x CUDA graph of 100 picks; the 16.8 MB store stays in L2 between picks"}


def run_c1_latency(dev):
    """Single-decision latency on C1 (1 queue x 8 requests, 16 bins): the
    pick kernel inside a CUDA graph of 100 launches, and the host round trip a
    serving scheduler would see (orloj_pick_batch_host: H2D of the queue,
    kernel, D2H of k*, stream synchronise), timed by the host clock over 2,000
    calls.  Context only: the paper times its CPU priority queue, not this
    (< 0.5 ms per insertion)."""
    import time

    import torch

    import gen
    import paper_2209_00159_b200 as orj
    import workloads as wl

    cfg = gen.config1()
    store = wl.score_store(cfg, dev)
    prof = wl.profile(cfg.profile)
    qs = wl.device_queues(cfg.queues, dev, with_arrival=False)
    bk = torch.empty(1, dtype=torch.int32, device=dev)
    bE = torch.empty(1, dtype=torch.float32, device=dev)
    stream = torch.cuda.Stream(dev)
    with torch.cuda.stream(stream):
        for _ in range(3):
            orj.pick_batch(store, prof, qs, bk, bE, stream)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=stream):
        for _ in range(100):
            orj.pick_batch(store, prof, qs, bk, bE, stream)
    with torch.cuda.stream(stream):
        g.replay()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(10):
            g.replay()
        e1.record(stream)
    torch.cuda.synchronize()
    graph_us = e0.elapsed_time(e1) * 1e3 / 1000
    q = cfg.queues
    pin = lambda a: torch.from_numpy(np.ascontiguousarray(a)).pin_memory()  # noqa: E731
    h_off, h_dl, h_dist, h_now = pin(q.offsets), pin(q.deadline), pin(q.dist), pin(q.now)
    from paper_2209_00159_b200 import _abi
    L = _abi.lib()
    need = L.orloj_pick_batch_host_workspace(1, int(q.offsets[-1]))
    wsb = torch.empty(need + 256, dtype=torch.uint8, device=dev)
    ws = (wsb.data_ptr() + 255) & ~255
    h_bk = torch.empty(1, dtype=torch.int32).pin_memory()
    h_bE = torch.empty(1, dtype=torch.float32).pin_memory()
    args = (store.c(), prof.c(), 1, h_off.data_ptr(), h_dl.data_ptr(), h_dist.data_ptr(), h_now.data_ptr(),
            h_bk.data_ptr(), h_bE.data_ptr(), ws, need, stream.cuda_stream)
    call = L.orloj_pick_batch_host
    for _ in range(20):
        _abi.check(call(*args))
        stream.synchronize()
    n = 2000
    t0 = time.perf_counter()
    for _ in range(n):
        call(*args)
        stream.synchronize()
    host_us = (time.perf_counter() - t0) / n * 1e6
    assert int(h_bk[0]) == int(bk.cpu()[0])
    return {"workload": "C1: 1 queue x 8 requests, 16 bins, kmax 8", "us_per_pick_in_graph": graph_us,
            "us_host_round_trip": host_us,
            "timing": "graph: 10 x CUDA graph of 100 picks (CUDA events); host: 2,000 x (orloj_pick_batch_host "
                      "called through ctypes + stream synchronise), host clock"}


MODEL_VARIANT_INSTR = os.path.join(ROOT, "profiles", "model_variants_instr.json")


def model_variant_specs(cfg, prof):
    """(name, duration table [kmax][B+1], interpolate, steps) of the C2 variants."""
    B = cfg.fam.B
    m = np.arange(B + 1, dtype=np.int64)
    logm = np.round(B * (2.0 ** (4.0 * m / B) - 1.0) / 15.0).astype(np.int64)
    tables = {"eq3": prof.a[:, None] + prof.w[:, None] * m[None, :],
              "log_grid": prof.a[:, None] + prof.w[:, None] * logm[None, :]}
    steps = ([-cfg.fam.p99_ticks() // 4, 0, cfg.fam.p99_ticks() // 2], [0.25, 1.0, 1.5])
    return [("eq3/edge/1 step", tables["eq3"], False, None), ("eq3/uniform/1 step", tables["eq3"], True, None),
            ("eq3/edge/3 steps", tables["eq3"], False, steps),
            ("log_grid/uniform/3 steps", tables["log_grid"], True, steps)]


def run_model_variants(dev, max_over_ranks, world):
    """Scoring-model variants on the C2 shape: 1,024
    SkipNet-like queues x 64, kmax 32, B 64 (orloj_score_model_batches, one
    launch per pick, 100 picks per CUDA graph).  Issue roofline per variant:
    the warp instructions of one launch (ncu, profiles/model_variants_instr.json,
    re-captured with scripts/gpu_model.sh whenever the model kernels change)
    over this run's time per pick, against the 148 x 4-scheduler issue peak."""
    import json

    import torch

    import gen
    import paper_2209_00159_b200 as orj
    import workloads as wl

    cfg = gen.config2()
    store = wl.score_store(cfg, dev)
    qs = wl.device_queues(cfg.queues, dev, with_arrival=False)
    prof = wl.profile(cfg.profile)
    Q = cfg.queues.Q
    instr = {}
    if os.path.exists(MODEL_VARIANT_INSTR):
        with open(MODEL_VARIANT_INSTR) as f:
            instr = json.load(f).get("instructions_per_launch", {})
    res = {}
    stream = torch.cuda.Stream(dev)
    for name, tab, interp, st in model_variant_specs(cfg, prof):
        model = orj.ScoreModel(tab, interpolate=interp, steps=st, device=dev)
        buf = {"E": torch.empty((Q, model.kmax), dtype=torch.float32, device=dev),
               "best_k": torch.empty(Q, dtype=torch.int32, device=dev),
               "best_E": torch.empty(Q, dtype=torch.float32, device=dev)}
        with torch.cuda.stream(stream):
            for _ in range(3):
                model.score(store, qs, stream, buf)
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=stream):
            for _ in range(100):
                model.score(store, qs, stream, buf)
        with torch.cuda.stream(stream):
            g.replay()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            for _ in range(10):
                g.replay()
            e1.record(stream)
        torch.cuda.synchronize()
        ms = max_over_ranks(e0.elapsed_time(e1)) / 1000
        res[name] = {"us_per_pick": 1e3 * ms, "decisions_per_s": world * Q / (ms / 1e3)}
        if name in instr:
            ach = instr[name] / (ms / 1e3) / 1e12
            peak = 148 * 4 * 1965e6 / 1e12
            res[name]["roofline"] = {"bound": "issue", "achieved": ach, "peak": peak, "unit": "T warp-instructions/s",
                                     "frac": ach / peak, "instructions_per_launch": instr[name],
                                     "instructions_source": "profiles/model_variants_instr.json (ncu)"}
    del store, qs
    return res


def run_priority(dev, max_over_ranks, world):
    """P1: one step = Eq. 1-2 log-priority of every queued
    request for every batch size 1..32 (orloj_priority_scores, [32][N] fp32
    out) + PopBatch of 32 per queue (orloj_pop_batch).  The per-size tables
    are built once, off the critical path, outside the timing."""
    import torch

    import gen
    import paper_2209_00159_b200 as orj
    import workloads as wl

    cfg = gen.config_priority()
    S = cfg.kmax
    store = wl.score_store(cfg, dev)
    prof = wl.profile(cfg.profile)
    qs = wl.device_queues(cfg.queues, dev, with_arrival=False)
    Q, N = cfg.queues.Q, cfg.queues.N
    tab = orj.PriorityTable(store, prof, S, 1.0 / cfg.fam.mean_ticks())
    lp = torch.empty((S, N), dtype=torch.float32, device=dev)
    bs = torch.full((Q,), S, dtype=torch.int32, device=dev)
    stream = torch.cuda.Stream(dev)
    with torch.cuda.stream(stream):
        for _ in range(3):
            tab.scores(qs, lp, stream)
            sel = tab.pop(qs, lp, bs, stream)
        iters = 20
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(2 * iters + 1)]
        ev[0].record(stream)
        for it in range(iters):
            tab.scores(qs, lp, stream)
            ev[2 * it + 1].record(stream)
            tab.pop(qs, lp, bs, stream, out=sel)
            ev[2 * it + 2].record(stream)
    torch.cuda.synchronize()
    ms_sc = max_over_ranks(sum(ev[2 * i].elapsed_time(ev[2 * i + 1]) for i in range(iters)) / iters)
    ms_pop = max_over_ranks(sum(ev[2 * i + 1].elapsed_time(ev[2 * i + 2]) for i in range(iters)) / iters)
    ms = ms_sc + ms_pop
    sc_bytes = N * (8 + 4 * S) + Q * (8 + 8)            # deadline in, S log p out; offsets, now
    pop_bytes = N * 4 + Q * (8 + 4 + 32 * 4)            # one size row in; offsets, bs, selection out
    peak, peak_src = measured_peaks()
    del store, qs, lp
    torch.cuda.empty_cache()
    return {"workload": "P1: Eq. 1-2 priorities, SkipNet-like 8-app mix (B 64), 65,536 queues x 256, "
                        "batch sizes 1..32, b = 1 / mean latency; PopBatch of 32 per queue",
            "requests": N, "sizes": S, "ms_per_step": ms, "ms_scores": ms_sc, "ms_pop": ms_pop,
            "scores_per_s": world * N * S / (ms / 1e3), "queues_per_s": world * Q / (ms / 1e3),
            "roofline_scores": {"bound": "hbm", "achieved": sc_bytes / (ms_sc / 1e3) / 1e9, "peak": peak,
                                "unit": "GB/s", "frac": sc_bytes / (ms_sc / 1e3) / 1e9 / peak,
                                "algorithmic_bytes_per_launch": sc_bytes, "peak_source": peak_src},
            "roofline_pop": {"bound": "hbm", "achieved": pop_bytes / (ms_pop / 1e3) / 1e9, "peak": peak,
                             "unit": "GB/s", "frac": pop_bytes / (ms_pop / 1e3) / 1e9 / peak,
                             "algorithmic_bytes_per_launch": pop_bytes},
            "timing": f"{iters} steps, CUDA events around each kernel on its stream"}


def build_replay(args, rank, world, dev):
    import gen
    import workloads as wl
    from paper_2209_00159_b200 import parallel

    nb = len(gen.BUCKET_SLO_MULTS)
    u = np.arange(nb * args.replay_seeds)
    mine = parallel.shard_round_robin(u // nb, rank, world)    # seed groups round-robin over ranks
    if getattr(args, "scenario_order", "seed") == "bucket":
        # the trace lists a rank's scenarios bucket by bucket: a block's warps then
        # replay scenarios of one SLO bucket (similar lengths), so fewer warp slots
        # idle while a block's slowest warp finishes (the counters are per bucket,
        # so the order changes nothing else)
        mine = mine[np.argsort(mine % nb, kind="stable")]
    return [wl.C5Family(name, local_ids=mine, n_arr=args.replay_arrivals, seeds_per_bucket=args.replay_seeds,
                        device=dev) for name in gen.C5_FAMILIES]


def family_segments(spec, name: str):
    """Per-family segment spec: "auto", an int, or "fam=G,...[,default]" (e.g.
    "rdi=16,auto"): the family's own entry, else the default (auto)."""
    spec = str(spec)
    if "=" not in spec:
        return spec
    default = "auto"
    for part in spec.split(","):
        if "=" in part:
            k, v = part.split("=", 1)
            if k.strip() == "last":    # time_replay: the family launched last
                continue
            if k.strip() == name:
                return v.strip()
        elif part.strip():
            default = part.strip()
    return default


def last_segments(spec, g: int, n_scen_family: int) -> int:
    """Segments of the family launched last: "last=G", "last=xM" (M times its
    own count) or "last=auto" in the spec, else its own count g.  "auto": 2x
    while the family has >= 2,048 scenarios on the rank (one GPU), else 4x
    (the shard sweeps of DESIGN.md §12: the last family's items set the drain)."""
    for part in str(spec).split(","):
        if "=" in part and part.split("=", 1)[0].strip() == "last":
            v = part.split("=", 1)[1].strip()
            if v == "auto":
                return g * (2 if n_scen_family >= 2048 else 4)
            return max(1, g * int(v[1:])) if v.startswith("x") else max(1, int(v))
    return g


def replay_segments(spec, n_scen_family: int, n_arr: int) -> int:
    """Segments per scenario for the segmented replay.  "auto": 8 per scenario
    while a family has >= 2,048 scenarios on this rank (the 1-GPU sweep), else 12
    (the 2/4/8-GPU shards; with the last family at 4x: DESIGN.md §12), never
    below ~2,000 arrivals per segment."""
    if spec != "auto":
        return max(1, int(spec))
    g = 8 if n_scen_family >= 2048 else 12
    return int(max(1, min(g, n_arr // 2000, 4096)))


REPLAY_LAUNCHES = os.path.join(ROOT, "profiles", "replay_sweep_launches.csv")


REPLAY_SWEEP_SEGS = [8, 8, 8, 16]   # the default sweep: 8 segments, 16 for the family launched last


def replay_sweep_instructions():
    """Warp instructions of one full 1-GPU C5 sweep at the default segments
    (REPLAY_SWEEP_SEGS): the sum of
    smsp__inst_executed.sum over the last sweep's launches in the committed
    ncu launch list (profiles/replay_sweep_launches.csv, re-captured with
    scripts/gpu_replay_check.sh whenever the replay kernel changes).  The
    count is a property of the deterministic workload and the code."""
    import csv
    if not os.path.exists(REPLAY_LAUNCHES):
        return None
    with open(REPLAY_LAUNCHES) as f:
        lines = [l for l in f if l.startswith('"')]
    rows = list(csv.reader(lines))
    h = rows[0]
    iI, iM, iV = h.index("ID"), h.index("Metric Name"), h.index("Metric Value")
    per = {}
    for r in rows[1:]:
        if r[iM] == "smsp__inst_executed.sum":
            per[int(r[iI])] = float(r[iV].replace(",", ""))
    ids = sorted(per)
    if len(ids) < 8:
        return None
    return int(sum(per[i] for i in ids[-8:]))      # one sweep = 4 families x 2 launches


def time_replay(fams, reps, dev, barrier, max_over_ranks, reduce=True, segments="auto"):
    """One sweep = the 4 family replays on 4 streams + one all-reduce of the
    [4 x 8 x 7] int64 counters (NCCL; a no-op on one rank), all inside the
    timed region.  Returns (ms per sweep, counters [4, 8, 7], clock summary)."""
    import torch

    import gen
    import paper_2209_00159_b200 as orj
    from paper_2209_00159_b200 import parallel

    nb = len(gen.BUCKET_SLO_MULTS)
    streams = [torch.cuda.Stream(dev) for _ in fams]
    main = torch.cuda.current_stream()
    tables = torch.zeros((len(fams), nb, 7), dtype=torch.int64, device=dev)
    segs = [replay_segments(family_segments(segments, f.tf.fam.name), f.trace.num_scenarios,
                            f.trace.num_arrivals // max(f.trace.num_scenarios, 1)) for f in fams]
    wss = [torch.empty(max(orj.replay_seg_workspace_bytes(f.trace, g), 1), dtype=torch.uint8, device=dev)
           for f, g in zip(fams, segs)]   # allocated once, outside the timed region

    order = list(range(len(fams)))

    def once():
        tables.zero_()
        start = torch.cuda.Event()
        start.record(main)
        for i in order:
            f, s, t_, g, ws = fams[i], streams[i], tables[i], segs[i], wss[i]
            s.wait_event(start)
            orj.replay_trace(f.store, f.profile, f.trace, per_bucket=t_, stream=s, segments=g, workspace=ws)
        for s in streams:
            ev = torch.cuda.Event()
            ev.record(s)
            main.wait_event(ev)
        if reduce:
            parallel.allreduce_counters(tables)

    once()  # warm-up
    torch.cuda.synchronize()
    # The second pass of a segmented replay (the stitch) is a latency-bound chain
    # per scenario that starts when the family's first pass ends.  Families whose
    # stitch re-ran the most decisions in the warm-up get the higher-priority
    # streams and are launched first, so their first pass finishes early and the
    # stitch overlaps the other families' first passes (independent work; the
    # counters do not depend on the order).
    if len(fams) > 1 and max(segs) > 1:
        work = [orj.replay_seg_stats(ws)["stitch_decisions"] if g > 1 else 0 for ws, g in zip(wss, segs)]
        order = sorted(range(len(fams)), key=lambda i: -work[i])
        lo, hi = torch.cuda.Stream.priority_range()       # (lowest, highest); numerically hi <= lo
        rank_of = {i: r for r, i in enumerate(order)}
        streams = [torch.cuda.Stream(dev, priority=min(lo, hi + rank_of[i])) for i in range(len(fams))]
        # The families run nearly one after another (stream priorities); the
        # sweep ends when the last family's first pass drains, which takes about
        # one of its items' duration.  "last=G" gives that family G segments
        # (shorter items) — chosen after the order is known, then re-warmed.
        lastg = last_segments(segments, segs[order[-1]], fams[order[-1]].trace.num_scenarios)
        if lastg != segs[order[-1]]:
            i = order[-1]
            segs[i] = lastg
            wss[i] = torch.empty(max(orj.replay_seg_workspace_bytes(fams[i].trace, lastg), 1), dtype=torch.uint8,
                                 device=dev)
            once()
            torch.cuda.synchronize()
    barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(dev.index) as clk:
        e0.record(main)
        for _ in range(reps):
            once()
        e1.record(main)
        torch.cuda.synchronize()
    barrier()
    time_replay.segments = segs
    time_replay.launch_order = [fams[i].tf.fam.name for i in order]
    time_replay.stats = [orj.replay_seg_stats(ws) if g > 1 else None for ws, g in zip(wss, segs)]
    return max_over_ranks(e0.elapsed_time(e1)) / reps, tables.cpu().numpy(), clk.summary()


def run_policies(args, rank, world, dev):
    """Replay policy variants (orloj_replay_trace_ex) on a
    smaller sweep: finish rate per family and SLO bucket for each
    (objective, drop rule); counters summed over ranks."""
    import torch

    import gen
    import paper_2209_00159_b200 as orj
    from paper_2209_00159_b200 import parallel, policy

    seeds = args.policy_seeds
    a2 = argparse.Namespace(**vars(args))
    a2.replay_seeds = seeds
    fams = build_replay(a2, rank, world, dev)
    thr = {f.tf.fam.name: torch.from_numpy(policy.expected_latency_thresholds(
        f.tf.fam.counts, f.tf.profile.a, f.tf.profile.w)).to(dev) for f in fams}
    nb = len(gen.BUCKET_SLO_MULTS)
    # segmented replay (same counters as the plain kernel, bit for bit), workspaces outside the timing
    segs = [replay_segments(family_segments(args.replay_segments, f.tf.fam.name), f.trace.num_scenarios,
                            args.replay_arrivals) for f in fams]
    wss = {f.tf.fam.name: torch.empty(max(orj.replay_seg_workspace_bytes(f.trace, g), 1), dtype=torch.uint8,
                                      device=dev) for f, g in zip(fams, segs)}
    out = {"sweep": f"4 families x 8 buckets x {seeds} seeds x {args.replay_arrivals} arrivals",
           "segments_per_scenario": segs}
    for objective in ("expected_finish", "finish_rate"):
        for drop in ("hopeless", "expected_latency"):
            tabs = torch.zeros((len(fams), nb, 7), dtype=torch.int64, device=dev)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for f, t_, g in zip(fams, tabs, segs):
                orj.replay_trace(f.store, f.profile, f.trace, per_bucket=t_, objective=objective,
                                 drop_threshold=thr[f.tf.fam.name] if drop == "expected_latency" else None,
                                 segments=g, workspace=wss[f.tf.fam.name])
            e1.record()
            parallel.allreduce_counters(tabs)
            torch.cuda.synchronize()
            c = tabs.cpu().numpy()
            out[f"{objective}/{drop}"] = {
                "ms": e0.elapsed_time(e1),
                "finish_rate_by_bucket": {f.tf.fam.name: [round(float(x), 4) for x in c[i, :, 1] / np.maximum(c[i, :, 0], 1)]
                                          for i, f in enumerate(fams)},
                "dropped_frac": round(float(c[:, :, 2].sum() / max(c[:, :, 0].sum(), 1)), 4)}
    # the paper's scheduler iteration (Alg. 1): per-size feasibility by E[L_bs] of the
    # all-application batch model, earliest-deadline candidate size, PopBatch by Eq. 1-2 priority
    tabs = torch.zeros((len(fams), nb, 7), dtype=torch.int64, device=dev)
    setup = []
    for f in fams:
        pt = orj.PriorityTable(f.store, f.profile, f.profile.kmax, 1.0 / f.tf.fam.mean_ticks())
        st = torch.from_numpy(policy.alg1_size_thresholds(f.tf.fam.counts, f.tf.profile.a, f.tf.profile.w)).to(dev)
        setup.append((pt, st))
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for f, t_, (pt, st), g in zip(fams, tabs, setup, segs):
        orj.replay_trace(f.store, f.profile, f.trace, per_bucket=t_, objective="alg1", priority=pt,
                         size_thresholds=st, segments=g, workspace=wss[f.tf.fam.name])
    e1.record()
    parallel.allreduce_counters(tabs)
    torch.cuda.synchronize()
    c = tabs.cpu().numpy()
    out["alg1 (Eq. 1-2 PopBatch, b = 1/mean)"] = {
        "ms": e0.elapsed_time(e1),
        "finish_rate_by_bucket": {f.tf.fam.name: [round(float(x), 4) for x in c[i, :, 1] / np.maximum(c[i, :, 0], 1)]
                                  for i, f in enumerate(fams)},
        "dropped_frac": round(float(c[:, :, 2].sum() / max(c[:, :, 0].sum(), 1)), 4)}
    return out


B_SWEEP_PER_MS = (1e-6, 1e-5, 1e-4, 1e-3, 1e-2, 1e-1)


def run_b_sweep(args, rank, world, dev):
    """Alg. 1 replay finish rate per SLO bucket as the anticipated-delay rate b
    of the Eq. 1-2 priority varies over 1e-6 .. 1e-1 per ms (PAPER.md:886-902,
    fig. eval-lambdas; the paper reports insensitivity, :623): the policy-sweep
    scenarios (32 seeds per bucket), segmented replay, counters summed over
    ranks.  The Eq. 2 tables are rebuilt per b (off the critical path)."""
    import torch

    import gen
    import paper_2209_00159_b200 as orj
    from paper_2209_00159_b200 import parallel, policy

    a2 = argparse.Namespace(**vars(args))
    a2.replay_seeds = args.policy_seeds
    fams = build_replay(a2, rank, world, dev)
    nb = len(gen.BUCKET_SLO_MULTS)
    segs = [replay_segments(family_segments(args.replay_segments, f.tf.fam.name), f.trace.num_scenarios,
                            args.replay_arrivals) for f in fams]
    wss = [torch.empty(max(orj.replay_seg_workspace_bytes(f.trace, g), 1), dtype=torch.uint8, device=dev)
           for f, g in zip(fams, segs)]
    thr = [torch.from_numpy(policy.alg1_size_thresholds(f.tf.fam.counts, f.tf.profile.a, f.tf.profile.w)).to(dev)
           for f in fams]
    out = {"sweep": f"4 families x 8 buckets x {args.policy_seeds} seeds x {args.replay_arrivals} arrivals, "
                    "Alg. 1 (Eq. 1-2 PopBatch)", "b_per_ms": list(B_SWEEP_PER_MS), "finish_rate_by_bucket": {},
           "ms": []}
    for b_ms in B_SWEEP_PER_MS:
        b = b_ms / 1000.0                     # 1 tick = 1 us
        tabs = torch.zeros((len(fams), nb, 7), dtype=torch.int64, device=dev)
        pts = [orj.PriorityTable(f.store, f.profile, f.profile.kmax, b) for f in fams]
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for f, t_, pt, st, g, ws in zip(fams, tabs, pts, thr, segs, wss):
            orj.replay_trace(f.store, f.profile, f.trace, per_bucket=t_, objective="alg1", priority=pt,
                             size_thresholds=st, segments=g, workspace=ws)
        e1.record()
        parallel.allreduce_counters(tabs)
        torch.cuda.synchronize()
        c = tabs.cpu().numpy()
        out["ms"].append(round(e0.elapsed_time(e1), 3))
        out["finish_rate_by_bucket"][f"{b_ms:g}"] = {
            f.tf.fam.name: [round(float(x), 4) for x in c[i, :, 1] / np.maximum(c[i, :, 0], 1)]
            for i, f in enumerate(fams)}
    rates = np.array([[v for fam in d.values() for v in fam] for d in out["finish_rate_by_bucket"].values()])
    out["max_spread_over_b"] = round(float((rates.max(0) - rates.min(0)).max()), 4)
    return out


FEEDBACK_EPOCHS, FEEDBACK_WINDOW, FEEDBACK_MIN, FEEDBACK_SAMPLE = 8, 2, 200, 0.125


def run_feedback(args, rank, world, dev):
    """Long-term feedback loop: the
    policy-sweep scenarios with an input drift half-way (half the
    applications 1.5x slower from epoch 4 of 8), replayed epoch by epoch
    (orloj_replay_feedback: profiler of 1/8 of the completed requests,
    refresh of rows with >= 200 window samples, window reset every 2
    epochs) against the same epochs with the static pre-drift store (no
    refresh).  Finish rate per epoch, all buckets pooled."""
    import torch

    import gen
    import paper_2209_00159_b200 as orj
    import workloads as wl
    from paper_2209_00159_b200 import parallel

    nb = len(gen.BUCKET_SLO_MULTS)
    u = np.arange(nb * args.policy_seeds)
    mine = parallel.shard_round_robin(u // nb, rank, world)
    E = FEEDBACK_EPOCHS
    res = {"workload": f"4 families x 8 buckets x {args.policy_seeds} seeds x {args.replay_arrivals} arrivals; "
                       f"drift at epoch {E // 2} of {E}", "epochs": E, "window_epochs": FEEDBACK_WINDOW,
           "min_samples": FEEDBACK_MIN, "sample_rate": FEEDBACK_SAMPLE, "finish_rate_by_epoch": {}, "ms": {}}
    for name in gen.C5_FAMILIES:
        if name == "static":
            continue                  # point masses: the drift only relabels the single bin
        f = wl.C5Family(name, local_ids=mine, n_arr=args.replay_arrivals, seeds_per_bucket=args.policy_seeds,
                        device=dev, drift=(E, E // 2))
        mask = wl.t(gen.sample_mask(gen.SEED_BASE + 41, f.trace.num_arrivals, FEEDBACK_SAMPLE), np.uint8, dev)
        rates = {}
        for mode, m in (("static", 1 << 31), ("feedback", FEEDBACK_MIN)):
            st = orj.HistogramStore.from_counts(f.tf.fam.counts, f.tf.fam.bin_ticks, dev)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            r = orj.replay_feedback(st, f.profile, f.trace, E, FEEDBACK_WINDOW, m, sample_mask=mask)
            e1.record()
            pe = r["per_epoch"]
            parallel.allreduce_counters(pe.view(-1, 7))
            torch.cuda.synchronize()
            c = pe.cpu().numpy().sum(1)            # [E][7], buckets pooled
            rates[mode] = [round(float(x), 4) for x in c[:, 1] / np.maximum(c[:, 0], 1)]
            res["ms"][f"{name}/{mode}"] = round(e0.elapsed_time(e1), 3)
        res["finish_rate_by_epoch"][name] = rates
        del f
    return res


def run_replay(args, rank, world, dev, barrier, max_over_ranks):
    import gen

    fams = build_replay(args, rank, world, dev)
    ms, tabs, clk = time_replay(fams, args.replay_reps, dev, barrier, max_over_ranks,
                                segments=args.replay_segments)
    segs = list(time_replay.segments)
    stitch = list(time_replay.stats)
    per_family = {f.tf.fam.name: t_ for f, t_ in zip(fams, tabs)}
    tot = tabs.sum(0)
    decisions = int(tot[:, 4].sum())
    arrivals = int(tot[:, 0].sum())
    assert (tot[:, 1] + tot[:, 2] + tot[:, 3] == tot[:, 0]).all()
    fr = {name: [round(float(x), 4) for x in (c[:, 1] / np.maximum(c[:, 0], 1))] for name, c in per_family.items()}
    util = {name: round(float(c[:, 5].sum() / max(c[:, 6].sum(), 1)), 4) for name, c in per_family.items()}
    out = {"workload": f"C5: 4 families x 8 SLO buckets x {args.replay_seeds} seeds x {args.replay_arrivals} "
                       f"arrivals (kmax 32, B 64), scenarios round-robin over {world} ranks",
           "value": decisions / (ms / 1e3), "unit": "decisions/s", "arrivals_per_s": arrivals / (ms / 1e3),
           "ms_per_sweep": ms, "decisions": decisions, "arrivals": arrivals, "scaling": "strong",
           "finish_rate_by_bucket": fr, "slo_multipliers": list(gen.BUCKET_SLO_MULTS), "utilisation": util,
           "segments_per_scenario": segs, "stitch_stats": stitch, "launch_order": list(time_replay.launch_order),
           "replay_kernel": "segmented (orloj_replay_trace_seg: speculative segments + stitch, 2 launches per family)"
                            if max(segs) > 1 else "plain (one warp per scenario)",
           "gpu_launches_per_sweep": sum(2 if g > 1 else 1 for g in segs), "clocks": clk,
           "collective": "one torch.distributed.all_reduce of the int64 [4 x 8 x 7] counters (NCCL) per sweep, "
                         "inside the timed region"}
    instr = replay_sweep_instructions()
    if (world == 1 and sorted(segs) == REPLAY_SWEEP_SEGS and args.replay_seeds == 256
            and args.replay_arrivals == 100_000 and instr):
        # issue roofline of the full 1-GPU sweep: the warp-instruction count is a
        # property of the (deterministic) workload and the code, counted by ncu
        # on the committed code (profiles/replay_sweep_launches.csv); the time is this run's
        peak = 148 * 4 * clk.get("sm_max_mhz", 1965) * 1e6 / 1e12     # 4 schedulers x 1 warp-instr/cycle per SM
        achieved = instr / (ms / 1e3) / 1e12
        out["roofline"] = {"bound": "issue", "achieved": achieved, "peak": peak, "unit": "T warp-instructions/s",
                           "frac": achieved / peak, "instructions_per_sweep": instr,
                           "instructions_per_decision": instr / max(decisions, 1),
                           "instructions_source": "profiles/replay_sweep_launches.csv (ncu smsp__inst_executed.sum)",
                           "peak_source": "148 SMs x 4 warp schedulers x 1 instruction/cycle at sm_max_mhz"}
    if not args.no_policies:
        with nvtx("policies"):
            out["policies"] = run_policies(args, rank, world, dev)
        with nvtx("b_sweep"):
            out["b_sweep"] = run_b_sweep(args, rank, world, dev)
        with nvtx("feedback"):
            out["feedback"] = run_feedback(args, rank, world, dev)
    if world == 1 and not args.no_shard_proxy:
        # strong-scaling proxy on one GPU: time EVERY rank's shard of an N-GPU run
        # (median of 3 sweeps each; everything but the ~10 us all-reduce) and take
        # the max over ranks, as a real N-GPU run would
        del fams
        out["shard_proxy"] = shard_proxy(args, dev, ms)
    return out


def shard_proxy(args, dev, ms_full):
    proxy = {"method": "each rank's round-robin shard replayed alone on this GPU, median of 3 sweeps; "
                       "implied speed-up = full sweep / max over ranks (not a measured N-GPU run)"}
    for N in (2, 4, 8):
        per_rank = []
        segs = None
        for r in range(N):
            sf = build_replay(args, r, N, dev)
            ts = []
            for _ in range(3):
                sms, _, _ = time_replay(sf, 1, dev, lambda: None, lambda x: x, reduce=False,
                                        segments=args.proxy_segments or args.replay_segments)
                ts.append(sms)
            per_rank.append(float(np.median(ts)))
            segs = list(time_replay.segments)
            del sf
        mx = max(per_rank)
        proxy[str(N)] = {"ms_per_rank": [round(x, 3) for x in per_rank], "ms_max_over_ranks": mx,
                         "ms_min_over_ranks": min(per_rank), "imbalance": mx / min(per_rank),
                         "implied_speedup": ms_full / mx, "segments_per_scenario": segs}
    return proxy


if __name__ == "__main__":
    main()
