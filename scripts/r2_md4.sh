timeout 1200 python -m pytest tests/test_gpu_mdlstm.py -q -x -p no:cacheprovider 2>&1 | tail -2
timeout 300 python scripts/mdlstm_bench.py 2>&1 | head -2
