"""Diagnostic: pinned host->device copy bandwidth and the e2e C3 pick time for
several chunk / stream counts (HostPicker)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import gen  # noqa: E402
import paper_2209_00159_b200 as orj  # noqa: E402
import workloads as wl  # noqa: E402


def bw(nbytes, reps=10):
    h = torch.empty(nbytes, dtype=torch.uint8).pin_memory()
    d = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
    d.copy_(h, non_blocking=True)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        d.copy_(h, non_blocking=True)
    e1.record()
    torch.cuda.synchronize()
    h2d = nbytes * reps / (e0.elapsed_time(e1) / 1e3) / 1e9
    e0.record()
    for _ in range(reps):
        h.copy_(d, non_blocking=True)
    e1.record()
    torch.cuda.synchronize()
    return h2d, nbytes * reps / (e0.elapsed_time(e1) / 1e3) / 1e9


def main():
    for nb in (16 << 20, 200 << 20):
        print(f"pinned copy {nb >> 20} MiB: H2D {bw(nb)[0]:.1f} GB/s, D2H {bw(nb)[1]:.1f} GB/s", flush=True)
    cfg = gen.config3()
    store = wl.c3_store(cfg)
    prof = wl.profile(cfg.profile)
    qn = cfg.queues
    h_off = torch.from_numpy(qn.offsets).pin_memory()
    h_dl = torch.from_numpy(qn.deadline).pin_memory()
    h_dist = torch.from_numpy(qn.dist).pin_memory()
    h_now = torch.from_numpy(qn.now).pin_memory()
    stream = torch.cuda.Stream()
    for chunks, streams in ((4, 2), (8, 2), (8, 3), (12, 2), (16, 2), (16, 3), (24, 2), (32, 3)):
        hp = orj.HostPicker(store, prof, qn.offsets, chunks=chunks, streams=streams)
        for _ in range(3):
            hp.pick(h_off, h_dl, h_dist, h_now, stream)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(stream):
            e0.record(stream)
            for _ in range(10):
                hp.pick(h_off, h_dl, h_dist, h_now, stream)
            e1.record(stream)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 10
        print(f"e2e chunks={chunks} streams={streams}: {ms:.3f} ms, {hp.h2d_bytes() / ms / 1e6:.1f} GB/s H2D", flush=True)
        del hp


if __name__ == "__main__":
    main()
