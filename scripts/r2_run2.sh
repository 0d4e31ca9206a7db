mkdir -p gpurun_out
export BLSTM_PARITY_LOG=$PWD/gpurun_out/r2_parity.jsonl; rm -f $BLSTM_PARITY_LOG
timeout 900 python -m pytest tests/test_gpu_fullsize_c5.py tests/test_gpu_fullsize.py tests/test_gpu_parity.py tests/test_gpu_step_mode.py tests/test_gpu_guards.py -q -s -p no:cacheprovider > gpurun_out/r2_t2.log 2>&1; tail -3 gpurun_out/r2_t2.log
nproc > gpurun_out/r2_cpu.txt; lscpu | grep "Model name" >> gpurun_out/r2_cpu.txt
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2_smoke_launches.csv python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2_smoke_ncu.log 2>&1; echo "ncu smoke rc=$?"
