timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
timeout 200 python tools/bench_parts.py 2>&1 | tail -4
python bench.py --config c4 --no-cpu-baseline 2>&1 | tail -1 | cut -c1-200
