O=gpurun_out/s3a; mkdir -p $O
timeout 600 python tools/slab_probe.py > $O/slab_probe.txt 2>&1
IRKG_GRAPHS=0 timeout 600 python tools/slab_probe.py > $O/slab_probe_nograph.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_multirank.py -x -q > $O/pytest_mr.log 2>&1; echo "exit $?" >> $O/pytest_mr.log
