mkdir -p gpurun_out
cat > /tmp/mdone.py <<'PY'
import os, sys
sys.path.insert(0, os.getcwd())
from scripts.mdlstm_bench import run
run(32, 256, 16, 16, 64, K=1)
PY
timeout 600 ncu --set full --import-source on -k regex:md_wave2 -c 2 -o gpurun_out/r2_md_wave2 -f python /tmp/mdone.py > gpurun_out/r2_md_ncu2.log 2>&1; echo ncu $?
ncu -i gpurun_out/r2_md_wave2.ncu-rep --page raw --csv > gpurun_out/r2_md2_raw.csv 2>/dev/null; echo raw $?
