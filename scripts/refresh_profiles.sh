#!/bin/bash
# Here (CPU box), after scripts/gpu_round2_final.sh: copy / summarise its gpurun_out/ into profiles/.
set -e
cd "$(dirname "$0")/.."
python scripts/ncu_summary.py full gpurun_out/prof_c3_pick.ncu-rep profiles/ncu_c3_pick_summary.json > /dev/null
python scripts/ncu_summary.py full gpurun_out/prof_replay.ncu-rep profiles/ncu_replay_seg_summary.json > /dev/null
python scripts/ncu_summary.py full gpurun_out/prof_c4.ncu-rep profiles/ncu_c4_small_summary.json > /dev/null
python scripts/ncu_summary.py full gpurun_out/prof_priority.ncu-rep /tmp/prio_full.json > /dev/null
python - <<'PY'
import json
d = json.load(open('/tmp/prio_full.json'))
for l in d['launches']:
    name = 'ncu_priority_scores_summary.json' if 'priority_scores' in l['kernel'] else 'ncu_pop_batch_summary.json'
    json.dump({"report": d['report'], "launches": [l], "dram_bytes_per_launch": l.get('dram_bytes_per_launch')},
              open('profiles/' + name, 'w'), indent=1)
PY
python scripts/ncu_summary.py launches gpurun_out/launches.csv profiles/r02_launches_c3_bench.json > /dev/null
cp gpurun_out/launches.csv profiles/r02_launches_c3_bench.csv
cp gpurun_out/bench.log profiles/r02_bench_full.log
cp gpurun_out/bench_ref.log profiles/r02_bench_reference.log
cp gpurun_out/parity_stats.jsonl profiles/r02_parity_stats.jsonl
cp gpurun_out/replay_sweep_launches.csv profiles/replay_sweep_launches.csv
cp gpurun_out/bench_priority.log profiles/r02_bench_priority.log
if [ -f gpurun_out/model_variants_instr.json ]; then
  sed 's#"source": "gpurun_out/model_launches.csv"#"source": "ncu launch list of scripts/model_variants_prof.py (scripts/gpu_round2_final.sh)"#' \
    gpurun_out/model_variants_instr.json > profiles/model_variants_instr.json
fi
[ -f gpurun_out/bench_n2_shared.log ] && cp gpurun_out/bench_n2_shared.log profiles/r02_bench_n2_shared_gpu_functional.log
echo refreshed
