for r in 1 2; do for v in u4c3 u3c4 u6c2 u2c6 u8c1 u5c2; do echo "== $v"; MHG_LIB=variants/libmhg_$v.so python profiles/conv_bench.py 16384 32768 2>&1 | tail -2; done; done
