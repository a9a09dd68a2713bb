"""Build a phase-timed copy of the replay kernel (clock64 at phase boundaries,
printed for the first scenarios) into build_variants/liborloj_phase.so.
Diagnostics only: never the product library."""
import os
import shutil
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
src = open(os.path.join(ROOT, "paper_2209_00159_b200/csrc/replay_kernel.cuh")).read()
marks = [
    ("  int64_t ndec = 0;\n", "  int64_t ndec = 0;\n  long long ph[8] = {0,0,0,0,0,0,0,0}; long long last = clock64(); "
     "long long nw1 = 0, nw2 = 0;\n#define PH(i) { __syncwarp(); long long now_ = clock64(); ph[i] += now_ - last; last = now_; }\n"),
    ("    // ---- 1. scan", "    PH(0)\n    // ---- 1. scan"),
    ("    while (wc < kmax) {", "    PH(1)\n    while (wc < kmax) {"),
    ("    if (wc == 0) continue;\n", "    PH(2)\n    if (wc == 0) continue;\n    if (wc == 1) ++nw1; else if (wc == 2) ++nw2;\n"),
    ("    const int mbin = ", "    PH(3)\n    const int mbin = "),
    ("    carry_off = kstar;\n    __syncwarp();\n  }\n", "    carry_off = kstar;\n    __syncwarp();\n    PH(4)\n  }\n"
     "  if (lane == 0 && s < 4) printf(\"PHASES s=%lld dec=%lld w1=%lld w2=%lld top=%lld carry=%lld arr=%lld "
     "score=%lld disp=%lld\\n\", (long long)s, (long long)ndec, nw1, nw2, ph[0], ph[1], ph[2], ph[3], ph[4]);\n"),
]
for a, b in marks:
    assert a in src, a
    src = src.replace(a, b, 1)
d = "/tmp/phase/csrc"
os.makedirs(d, exist_ok=True)
for f in ("common.cuh", "score_kernel.cuh", "store_kernel.cuh", "orloj.cu"):
    shutil.copy(os.path.join(ROOT, "paper_2209_00159_b200/csrc", f), d)
open(os.path.join(d, "replay_kernel.cuh"), "w").write(src)
cu = open(os.path.join(d, "orloj.cu")).read().replace('"../../include/orloj.h"', f'"{ROOT}/include/orloj.h"')
open(os.path.join(d, "orloj.cu"), "w").write(cu)
subprocess.check_call(["nvcc", "-O3", "-std=c++17", "-gencode", "arch=compute_100a,code=sm_100a", "-lineinfo",
                       *sys.argv[1:], "-shared", "-Xcompiler", "-fPIC", "-o",
                       os.path.join(ROOT, "build_variants/liborloj_phase.so"), os.path.join(d, "orloj.cu")])
