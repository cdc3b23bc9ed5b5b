python tools/debug_fast.py 300 2>&1 | tail -5
python tools/debug_fast.py 65536 big 2>&1 | tail -5
