import os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2209_00159_b200 as orj
import workloads as wl
for fam in ("skipnet", "rdi", "gpt", "static"):
    f = wl.C5Family(fam, local_ids=np.arange(4), n_arr=100000)
    orj.replay_trace(f.store, f.profile, f.trace)
    torch.cuda.synchronize()
    print("family", fam, flush=True)
