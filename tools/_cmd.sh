timeout 900 python -m pytest tests -q -x -m gpu -k "large or c3 or any_n or uniform" 2>&1 | tail -2
python bench.py --config c3 --no-cpu-baseline 2>&1 | tail -1 | cut -c1-200
