import sys; sys.path.insert(0,'/root/repo'); sys.path.insert(0,'/root/repo/tests')
import numpy as np, torch
import test_gpu_priority as T
from oracle import priority as pr
import gen
fam, prof, q = T._case("gpt", gen.SEED_BASE + 920, Q=64)
b = 1.0 / fam.mean_ticks(); p99 = fam.p99_ticks()
offs, costs = [-p99 // 4, 0, p99 // 2], [0.25, 1.0, 1.75]
tab, qs, _ = T._gpu_scores(fam, prof, q, b)
lp = tab.scores(qs, steps=(offs, costs)); torch.cuda.synchronize()
got = lp.cpu().numpy().T.astype(np.float64)
ref = pr.scores_steps(fam.counts, prof.a, prof.w, T.S, b, q.offsets, q.deadline, q.now, offs, costs, store_fp32=True)
fin = np.isfinite(ref)
err = np.where(fin, np.abs(got - ref), 0)
j, k = np.unravel_index(np.argmax(err), err.shape)
qi = np.searchsorted(q.offsets, j, side='right') - 1
sig = int(q.deadline[j] - q.now[qi])
print("j", j, "k", k + 1, "sigma", sig, "got", got[j, k], "ref", ref[j, k], "b", b, "p99", p99)
pm = pr.batch_latency_pmf(fam.counts, k + 1, store_fp32=True)
for o in offs:
    print(" off", o, "single", pr.log_priority(pm, float(prof.a[k]), float(prof.w[k]), b, [sig + o])[0])
sing = tab.scores(qs).cpu().numpy().T
print("gpu single at 0:", sing[j, k])
print("a,w", prof.a[k], prof.w[k], "B", fam.B, "horizon", prof.a[k] + prof.w[k] * fam.B)
