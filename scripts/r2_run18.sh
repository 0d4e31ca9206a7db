cp paper_1608_00895_b200/libblstm.so /tmp/prod.so; cp build/libblstm_trace.so paper_1608_00895_b200/libblstm.so
for B in 81 40 20; do echo "== B=$B"; timeout 200 python scripts/trace_rec.py --B $B 2>&1 | grep -E "median|wait|MMA|gate|send|stores|TMEM|cell|gather|dA|P " ; done
cp /tmp/prod.so paper_1608_00895_b200/libblstm.so
