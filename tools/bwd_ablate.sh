for d in 8 9 40 72 12; do echo "== TTB_DBG=$d"; TTB_DBG=$d python tools/bwd_stamps.py cfg2 | head -10; done
