#!/bin/bash
# One GPU-box pass: parity tests, smoke, bench, ncu launch list + one full capture.
# Usage (from the repo root, through gpurun): bash tools/gpu_check.sh TAG
TAG=${1:-run}
O=gpurun_out/$TAG
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $O/smi.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "pytest exit $?" >> $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke exit $?" >> $O/smoke.log
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err; echo "bench exit $?" >> $O/bench.err
if [ "${SKIP_NCU:-0}" != "1" ]; then
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu > $O/ncu_launch.log 2>&1; echo "ncu exit $?" >> $O/ncu_launch.log
python tools/launch_summary.py $O/launches.csv > $O/launch_summary.txt 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_cgs -s 400 -c 6 \
  -o $O/cgs_full python bench.py --steps 1 --warmup 3 --no-cpu > $O/ncu_full.log 2>&1; echo "ncu full exit $?" >> $O/ncu_full.log
fi
tail -3 $O/*.log $O/bench.err
