mkdir -p gpurun_out
export BLSTM_PARITY_LOG=$PWD/gpurun_out/r2_parity17.jsonl; rm -f $BLSTM_PARITY_LOG
timeout 1500 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/r2_t17.log 2>&1; tail -3 gpurun_out/r2_t17.log
unset BLSTM_PARITY_LOG
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2_smoke17.log 2>&1; echo smoke $?
timeout 400 python bench.py --steps 20 --warmup 5 > gpurun_out/r2_b17_c3.log 2>&1; tail -1 gpurun_out/r2_b17_c3.log | cut -c1-200
