mkdir -p gpurun_out
export BLSTM_PARITY_LOG=$PWD/gpurun_out/r2_parity9.jsonl; rm -f $BLSTM_PARITY_LOG
timeout 900 python -m pytest tests/test_gpu_step_mode.py tests/test_gpu_fullsize_c5.py -q -x -p no:cacheprovider > gpurun_out/r2_t9.log 2>&1; tail -3 gpurun_out/r2_t9.log
cp paper_1608_00895_b200/libblstm.so /tmp/libblstm_prod.so
cp build/libblstm_trace.so paper_1608_00895_b200/libblstm.so
timeout 300 python scripts/trace_rec.py --config C5 > gpurun_out/r2_trace9_c5.txt 2>&1; grep -A12 "backward" gpurun_out/r2_trace9_c5.txt
cp /tmp/libblstm_prod.so paper_1608_00895_b200/libblstm.so
for v in "" "BLSTM_STEP_PERSIST_BWD=0"; do env $v timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --config C5 > gpurun_out/r2_b9.log 2>&1; echo "$v"; tail -1 gpurun_out/r2_b9.log | python -c "import json,sys; j=json.loads(sys.stdin.read()); print(round(j['value']), j['ms_per_step'], j['kernel_ms_per_step'])"; done
timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/r2_b9_c3.log 2>&1; tail -1 gpurun_out/r2_b9_c3.log | python -c "import json,sys; j=json.loads(sys.stdin.read()); print('C3', round(j['value']), j['ms_per_step'], j['kernel_ms_per_step'])"
