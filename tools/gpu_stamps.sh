python tools/bwd_stamps.py cfg2 2>&1 | tail -12
