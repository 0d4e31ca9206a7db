# A/B of library builds at C5: bash scripts/ab_c5.sh build/libA.so build/libB.so ... (3 rounds, one bench line each)
for r in 1 2 3; do
  for so in "$@"; do
    cp $so paper_1608_00895_b200/libblstm.so
    timeout 400 python bench.py --steps 3 --warmup 3 --config C5 --no-cpu-baseline > gpurun_out/ab_c5.log 2>&1
    tail -1 gpurun_out/ab_c5.log | python -c "import json,sys; j=json.loads(sys.stdin.read()); k=j.get('kernel_ms_per_step'); print('$so', round(j['value']), round(j['ms_per_step'],3), round(k['lstm_rec_fwd'],2), round(k['lstm_rec_bwd'],2), j['clocks']['sm_mhz'])" 2>&1 | tail -1
  done
done
cp $1 paper_1608_00895_b200/libblstm.so
