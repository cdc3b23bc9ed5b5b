# config-3 backward ablations (event times): TTB_DBG 1 = no dG3 reductions, 4 = no dG1/dG2 reductions
for d in 0 1 4 5; do echo "== TTB_DBG=$d"; if [ $d = 0 ]; then python tools/cfg_kernels.py cfg3; else TTB_DBG=$d python tools/cfg_kernels.py cfg3; fi; done
TTB_DBG=8 python tools/bwd_stamps.py cfg3
