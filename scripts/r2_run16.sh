mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_mdlstm.py -q -x -p no:cacheprovider 2>&1 | tail -2
timeout 300 python scripts/mdlstm_bench.py 2>&1 | head -2
cp paper_1608_00895_b200/libblstm.so /tmp/cur.so
bash scripts/ab_bench.sh fk "" build/libblstm_fork.so build/libblstm_new.so
cp /tmp/cur.so paper_1608_00895_b200/libblstm.so
