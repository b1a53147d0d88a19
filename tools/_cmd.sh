timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
timeout 200 python tools/bench_parts.py 2>&1 | tail -4 | head -2
timeout 120 python tools/dbg_resample.py 2>&1 | tail -3
