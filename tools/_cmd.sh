timeout 900 python -m pytest tests -q -x -m gpu 2>&1 | tail -2
python bench.py --config c4 --no-cpu-baseline 2>&1 | tail -1 | cut -c1-200
