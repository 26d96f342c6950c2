O=gpurun_out/s3c; mkdir -p $O
for b in 1 4 8; do echo "== batch $b"; IRKG_SLAB_BATCH=$b timeout 600 python tools/slab_probe.py 2>&1 | grep -v NCCL; done > $O/slab_probe.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_multirank.py -x -q > $O/pytest.log 2>&1; echo "exit $?" >> $O/pytest.log
