timeout 600 python bench.py --config e1 --steps 10 --warmup 3 2>&1 | tail -1
timeout 600 python bench.py --impl reference --config e1 --steps 5 --warmup 1 2>&1 | tail -1
