mkdir -p gpurun_out
export BLSTM_PARITY_LOG=$PWD/gpurun_out/r2_parity13.jsonl; rm -f $BLSTM_PARITY_LOG
timeout 1500 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/r2_t13.log 2>&1; tail -3 gpurun_out/r2_t13.log
unset BLSTM_PARITY_LOG
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2_smoke13.log 2>&1; echo smoke $?
timeout 400 python bench.py --steps 20 --warmup 5 > gpurun_out/r2_b13_c3.log 2>&1; tail -1 gpurun_out/r2_b13_c3.log | python -c "import json,sys; j=json.loads(sys.stdin.read()); print('C3', round(j['value']), j['ms_per_step'], j['kernel_ms_per_step'])"
timeout 400 python bench.py --steps 3 --warmup 3 --config C5 --no-cpu-baseline > gpurun_out/r2_b13_c5.log 2>&1; tail -1 gpurun_out/r2_b13_c5.log | python -c "import json,sys; j=json.loads(sys.stdin.read()); print('C5', round(j['value']), j['ms_per_step'], j['kernel_ms_per_step'])"
timeout 300 python scripts/gemm_bench.py > gpurun_out/r2_gemm_bench.txt 2>&1; cat gpurun_out/r2_gemm_bench.txt
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r2_launches13_c3.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/r2_ncu13.log 2>&1; echo ncu $?
