mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r2_smi.txt
timeout 1500 python -m pytest tests -m gpu -q -s -p no:cacheprovider > gpurun_out/r2_t1.log 2>&1; tail -5 gpurun_out/r2_t1.log
timeout 300 python bench.py --steps 20 --warmup 5 > gpurun_out/r2_b1.log 2>&1; tail -1 gpurun_out/r2_b1.log | cut -c1-600
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2_smoke.log 2>&1; echo smoke $?
