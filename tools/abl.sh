for d in 0 1 2 3 4 7; do echo "dbg=$d"; TTB_DBG=$d python tools/check_fast.py 2>&1 | grep -A2 "det=False" | grep -E "f_bwd|det=False"; done
