# persistent BPTT: parity (KS 4 / 8 at Hq 512), C5 trace with the MMA-only / load-only experiments
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_step_mode.py -q -p no:cacheprovider -k "persistent_bptt" > gpurun_out/pb_tests.log 2>&1; tail -3 gpurun_out/pb_tests.log
cp paper_1608_00895_b200/libblstm.so /tmp/main.so
cp build/libblstm_trace.so paper_1608_00895_b200/libblstm.so
for e in 0 1 2; do
  BLSTM_PB_EXP=$e timeout 300 python scripts/trace_rec.py --config C5 > gpurun_out/pb_trace_e$e.txt 2>&1; echo exp $e; sed -n '/^backward/,$p' gpurun_out/pb_trace_e$e.txt
done
cp /tmp/main.so paper_1608_00895_b200/libblstm.so
