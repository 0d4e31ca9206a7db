mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -q -x -p no:cacheprovider > gpurun_out/r2_t19.log 2>&1; tail -3 gpurun_out/r2_t19.log
for v in "" "BLSTM_FWD_SPLIT=0" "" "BLSTM_FWD_SPLIT=0"; do env $v timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/r2_b19.log 2>&1; echo "$v"; tail -1 gpurun_out/r2_b19.log | python -c "import json,sys; j=json.loads(sys.stdin.read()); print(round(j['value']), j['ms_per_step'], {k: round(v,3) for k,v in j['kernel_ms_per_step'].items()})" 2>&1 | tail -1; done
cp paper_1608_00895_b200/libblstm.so /tmp/prod.so; cp build/libblstm_trace.so paper_1608_00895_b200/libblstm.so
timeout 200 python scripts/trace_rec.py 2>&1 | head -16
cp /tmp/prod.so paper_1608_00895_b200/libblstm.so
