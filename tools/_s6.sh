O=gpurun_out/s6; mkdir -p $O
for r in 0 2 5 1 4; do IRKG_CGS_REV=$r timeout 600 python bench.py --no-cpu > $O/bench_rev$r.json 2>$O/bench_rev$r.err; done
timeout 900 python -m pytest tests -m gpu -x -q > $O/pytest.log 2>&1; echo "exit $?" >> $O/pytest.log
