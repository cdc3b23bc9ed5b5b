# config-2 backward ablations (event times): TTB_DBG 1 = no dG3 reductions, 4 = no dG1/dG2 reductions,
# 32 = no per-lookup FMA work, 64 = no per-lookup loop at all
for d in 0 1 4 32 64 97; do echo "== TTB_DBG=$d"; if [ $d = 0 ]; then python tools/cfg_kernels.py cfg2; else TTB_DBG=$d python tools/cfg_kernels.py cfg2; fi; done 2>&1 | grep -v Warn
