#!/bin/bash
# One GPU-box pass: parity tests, smoke, bench, ncu launch list + full captures.
# Usage (from the repo root, through gpurun): bash tools/gpu_check.sh TAG
TAG=${1:-run}
O=gpurun_out/$TAG
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $O/smi.txt 2>&1
if [ "${SKIP_TESTS:-0}" != "1" ]; then
timeout 1500 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "pytest exit $?" >> $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke exit $?" >> $O/smoke.log
fi
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err; echo "bench exit $?" >> $O/bench.err
timeout 600 python tools/phase_probe.py > $O/probe.txt 2>&1
if [ "${SKIP_NCU:-0}" != "1" ]; then
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu --no-large > $O/ncu_launch.log 2>&1; echo "ncu exit $?" >> $O/ncu_launch.log
python tools/launch_summary.py $O/launches.csv > $O/launch_summary.txt 2>&1
# CGS sweeps at a pinned Arnoldi index (j = 8): per-launch DRAM traffic vs algorithmic bytes
timeout 900 ncu --set full --clock-control none --import-source on --nvtx --nvtx-include "probe6/" -k regex:k_cgs -s 6 -c 3 \
  -o $O/cgs_j8 python tools/phase_probe.py --js 8 --reps 2 > $O/ncu_cgs.log 2>&1; echo "ncu cgs exit $?" >> $O/ncu_cgs.log
timeout 900 ncu --set full --clock-control none --import-source on --nvtx --nvtx-include "probe8/" -k regex:"k_jacobi_sp2d|k_block_op_strip" -s 6 -c 3 \
  -o $O/stencil_full python tools/phase_probe.py --js 4 --reps 2 > $O/ncu_stencil.log 2>&1; echo "ncu stencil exit $?" >> $O/ncu_stencil.log
python tools/ncu_summary.py $O/cgs_j8.ncu-rep > $O/cgs_j8_summary.csv 2>&1
python tools/ncu_summary.py $O/stencil_full.ncu-rep > $O/stencil_summary.csv 2>&1
fi
tail -n 3 $O/*.log $O/bench.err
