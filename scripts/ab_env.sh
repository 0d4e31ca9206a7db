# A/B of environment settings at C3 (same library): bash scripts/ab_env.sh "ENV_A" "ENV_B" ... (3 rounds)
for r in 1 2 3; do
  for e in "$@"; do
    env $e timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/ab_env.log 2>&1
    tail -1 gpurun_out/ab_env.log | python -c "import json,sys; j=json.loads(sys.stdin.read()); print('$e', round(j['value']), round(j['ms_per_step'],4), {k: round(v,3) for k,v in j['kernel_ms_per_step'].items()})" 2>&1 | tail -1
  done
done
