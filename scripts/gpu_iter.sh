#!/bin/bash
# One measurement iteration on the GPU box: parity tests, a bench line, and the per-step phase
# trace of the recurrence kernels.  Usage: bash scripts/gpu_iter.sh TAG   (outputs gpurun_out/*TAG*)
tag=${1:-x}
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/t_$tag.log 2>&1; tail -2 gpurun_out/t_$tag.log
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/b_$tag.log 2>&1
python - "$tag" <<'PY'
import json, sys
l = [x for x in open(f"gpurun_out/b_{sys.argv[1]}.log") if x.startswith("{")]
if l:
    j = json.loads(l[-1])
    print("value", round(j["value"]), "ms/step", round(j["ms_per_step"], 3), "kernels", {k: round(v, 3) for k, v in j["kernel_ms_per_step"].items()})
else:
    print(open(f"gpurun_out/b_{sys.argv[1]}.log").read()[-2000:])
PY
python paper_1608_00895_b200/csrc/build.py --trace --force > /dev/null && timeout 300 python scripts/trace_rec.py > gpurun_out/trace_$tag.txt 2>&1; cat gpurun_out/trace_$tag.txt
python paper_1608_00895_b200/csrc/build.py --force > /dev/null
