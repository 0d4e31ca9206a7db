mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_mdlstm.py -q -x -s -p no:cacheprovider > gpurun_out/r2_md_t.log 2>&1; grep -E "passed|failed|parity|Error" gpurun_out/r2_md_t.log | tail -40
timeout 300 python scripts/mdlstm_bench.py > gpurun_out/r2_md_bench.txt 2>&1; cat gpurun_out/r2_md_bench.txt
cp paper_1608_00895_b200/libblstm.so /tmp/prod.so; cp build/libblstm_trace.so paper_1608_00895_b200/libblstm.so
timeout 120 python scripts/trace_md.py --H 64
cp /tmp/prod.so paper_1608_00895_b200/libblstm.so
