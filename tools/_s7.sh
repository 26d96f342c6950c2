O=gpurun_out/s7; mkdir -p $O
timeout 900 python -m pytest tests -m gpu -x -q > $O/pytest.log 2>&1; echo "exit $?" >> $O/pytest.log
timeout 300 python tools/phase_probe.py --js 4 > $O/probe.txt 2>&1
timeout 600 python bench.py --no-cpu > $O/bench.json 2>$O/bench.err
