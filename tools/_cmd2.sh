timeout 200 python tools/phase_timing.py 2>&1 | tail -24
