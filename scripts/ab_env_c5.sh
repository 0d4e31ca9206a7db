# A/B of environment settings at C5 (same library): bash scripts/ab_env_c5.sh "ENV_A" "ENV_B" ... (3 rounds)
for r in 1 2 3; do
  for e in "$@"; do
    env $e timeout 400 python bench.py --steps 3 --warmup 3 --config C5 --no-cpu-baseline > gpurun_out/ab_env_c5.log 2>&1
    tail -1 gpurun_out/ab_env_c5.log | python -c "import json,sys; j=json.loads(sys.stdin.read()); k=j['kernel_ms_per_step']; print('$e', round(j['value']), round(j['ms_per_step'],3), {a: round(b,2) for a,b in k.items()}, j['clocks']['sm_mhz'])" 2>&1 | tail -1
  done
done
