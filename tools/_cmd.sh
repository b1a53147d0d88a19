for v in base rcp3 sqrt3 ones all3 base all3; do echo $v; CVA_LIB_PATH=build/var_$v.so timeout 200 python tools/bench_parts.py 2>&1 | tail -4 | head -2; done
CVA_LIB_PATH=build/var_all3.so timeout 120 python tools/dbg_resample.py 2>&1 | tail -6
CVA_LIB_PATH=build/var_all3.so timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
