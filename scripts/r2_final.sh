mkdir -p gpurun_out
export BLSTM_PARITY_LOG=$PWD/gpurun_out/r2_parity_final.jsonl; rm -f $BLSTM_PARITY_LOG
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider -rs > gpurun_out/r2_tests_final.log 2>&1; tail -3 gpurun_out/r2_tests_final.log
unset BLSTM_PARITY_LOG
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2_smoke_final.log 2>&1; echo smoke $?; tail -2 gpurun_out/r2_smoke_final.log
timeout 400 python bench.py --steps 20 --warmup 5 > gpurun_out/r2_bench_c3_final.log 2>&1; tail -1 gpurun_out/r2_bench_c3_final.log | cut -c1-250
timeout 400 python bench.py --steps 3 --warmup 3 --config C5 > gpurun_out/r2_bench_c5_final.log 2>&1; tail -1 gpurun_out/r2_bench_c5_final.log | cut -c1-250
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/r2_bench_ref_final.log 2>&1; tail -1 gpurun_out/r2_bench_ref_final.log | cut -c1-250
timeout 300 python scripts/mdlstm_bench.py > gpurun_out/r2_md_bench_final.txt 2>&1
timeout 300 python scripts/gemm_bench.py > gpurun_out/r2_gemm_bench_final.txt 2>&1
timeout 300 python scripts/timeline.py > gpurun_out/r2_timeline_final.txt 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r2_launches_final_c3.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/r2_ncu_final.log 2>&1; echo ncu $?
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2_smoke_launches_final.csv python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2_ncu_smoke_final.log 2>&1; echo ncu_smoke $?
