#!/bin/bash
# A/B sweep of engine tuning knobs on the bench workload and the phase probe.
# Usage (through gpurun): bash tools/env_sweep.sh TAG "ENV1=a ENV2=b" "ENV1=c" ...
TAG=$1; shift
O=gpurun_out/$TAG
mkdir -p $O
i=0
for cfg in "" "$@"; do
  echo "=== [$cfg]" >> $O/sweep.txt
  env $cfg timeout 300 python bench.py --no-cpu > $O/b$i.json 2> $O/b$i.err
  python - $O/b$i.json >> $O/sweep.txt <<'PY'
import json, sys
d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
r = d["roofline"]
print(f"ms/step {d['ms_per_step']:.2f}  value {d['value']/1e9:.4f} G  cgs {r['achieved']:.0f} GB/s avg {r['avg_launch_us']:.1f} us  e2e {d['e2e']['value']/1e9:.4f} G  kry {d['krylov_iterations']}")
PY
  env $cfg timeout 300 python tools/phase_probe.py --reps 30 --js 0,4,8,16,32 > $O/p$i.txt 2>&1
  grep -E "^ +[0-9]+ " $O/p$i.txt >> $O/sweep.txt
  i=$((i+1))
done
cat $O/sweep.txt
