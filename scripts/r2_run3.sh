mkdir -p gpurun_out
export BLSTM_PARITY_LOG=$PWD/gpurun_out/r2_parity3.jsonl; rm -f $BLSTM_PARITY_LOG
timeout 900 python -m pytest tests/test_gpu_fullsize_c5.py tests/test_gpu_fullsize.py tests/test_gpu_parity.py tests/test_gpu_guards.py -q -s -p no:cacheprovider > gpurun_out/r2_t3.log 2>&1; tail -3 gpurun_out/r2_t3.log
for p in fp16 fp16x2w; do timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --precision $p > gpurun_out/r2_b3_$p.log 2>&1; tail -1 gpurun_out/r2_b3_$p.log | cut -c1-250; done
timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --config C5 --precision fp16x2w > gpurun_out/r2_b3_c5x2w.log 2>&1; tail -1 gpurun_out/r2_b3_c5x2w.log | cut -c1-250
