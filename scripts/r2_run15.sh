mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/r2_t15.log 2>&1; tail -3 gpurun_out/r2_t15.log
timeout 400 python bench.py --steps 20 --warmup 5 > gpurun_out/r2_b15_c3.log 2>&1; tail -1 gpurun_out/r2_b15_c3.log | python -c "import json,sys; j=json.loads(sys.stdin.read()); print('C3', round(j['value']), j['ms_per_step'], j['kernel_ms_per_step'])"
timeout 400 python bench.py --steps 3 --warmup 3 --config C5 --no-cpu-baseline > gpurun_out/r2_b15_c5.log 2>&1; tail -1 gpurun_out/r2_b15_c5.log | python -c "import json,sys; j=json.loads(sys.stdin.read()); print('C5', round(j['value']), j['ms_per_step'], j['kernel_ms_per_step'])"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r2_launches15_c3.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/r2_ncu15.log 2>&1; echo ncu $?
