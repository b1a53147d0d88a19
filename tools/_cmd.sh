timeout 900 python -m pytest tests -q -x -m gpu -k "allpairs or c2" 2>&1 | tail -2
python bench.py --config c2 --no-cpu-baseline 2>&1 | tail -1 | cut -c1-200
