cp build/libblstm_trace.so /tmp/tr.so; cp paper_1608_00895_b200/libblstm.so /tmp/prod.so
cp /tmp/tr.so paper_1608_00895_b200/libblstm.so
timeout 120 python scripts/trace_md.py --H 64
timeout 120 python scripts/trace_md.py --H 32
cp /tmp/prod.so paper_1608_00895_b200/libblstm.so
