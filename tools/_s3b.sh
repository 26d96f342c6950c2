O=gpurun_out/s3b; mkdir -p $O
timeout 600 python tools/slab_probe.py > $O/slab_probe.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > $O/pytest.log 2>&1; echo "exit $?" >> $O/pytest.log
