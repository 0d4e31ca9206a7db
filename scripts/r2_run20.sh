bash scripts/ab_bench.sh ns "" build/libblstm_base.so build/libblstm_nostore.so 2>&1 | head -4
