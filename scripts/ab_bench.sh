# A/B of library builds: bash scripts/ab_bench.sh TAG "extra bench args" build/libA.so build/libB.so ...
# alternates the builds (3 rounds), one C3 bench line each; restores the first build at the end
tag=$1; args=$2; shift 2
for r in 1 2 3; do
  for so in "$@"; do
    cp $so paper_1608_00895_b200/libblstm.so
    timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline $args > gpurun_out/ab_$tag.log 2>&1
    tail -1 gpurun_out/ab_$tag.log | python -c "import json,sys; j=json.loads(sys.stdin.read()); print('$so', round(j['value']), round(j['ms_per_step'],4), {k: round(v,3) for k,v in j['kernel_ms_per_step'].items()})" 2>&1 | tail -1
  done
done
cp $1 paper_1608_00895_b200/libblstm.so
