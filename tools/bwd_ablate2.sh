for d in 0 1 4 5; do TTB_DBG=$d python tools/cfg_kernels.py cfg2 | sed "s/^/dbg=$d /"; done
