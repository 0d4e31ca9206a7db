mkdir -p gpurun_out
bash scripts/ab_bench.sh sc "" build/libblstm_new.so build/libblstm_old.so
timeout 300 python scripts/timeline.py > gpurun_out/r2_timeline14.txt 2>&1; tail -60 gpurun_out/r2_timeline14.txt
