timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py tests/test_gpu_dropout.py -q -x -p no:cacheprovider 2>&1 | tail -2
bash scripts/ab_bench.sh pt "" build/libblstm_ptr.so build/libblstm_base.so
