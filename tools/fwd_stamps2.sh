for d in ${DBGS:-16 48 80 112}; do echo "dbg=$d"; TTB_DBG=$d python tools/fwd_stamps.py 2>&1 | tail -6 | python -c "
import sys,re
rows=[list(map(int,re.findall(r'-?\d+',l))) for l in sys.stdin.read().strip().split('\n')[1:]]
import numpy as np
r=np.array(rows); print('loads', r[1]-r[0], 'mma', r[2]-r[1], 'epi', r[4]-r[2], 'endsync', r[3]-r[4])"; done
