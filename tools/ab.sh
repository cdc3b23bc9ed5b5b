# A/B kernel timing: ab/libttb_base.so (a baseline build) against the tree's libttb.so
# usage: bash tools/ab.sh [workloads...]   (default: cfg2 cfg3)
wls=${@:-cfg2 cfg3}
for r in 1 2; do
  for wl in $wls; do
    echo "base $(TTB_LIB_PATH=ab/libttb_base.so timeout 300 python tools/cfg_kernels.py $wl 2>&1 | tail -1)"
    echo "new  $(timeout 300 python tools/cfg_kernels.py $wl 2>&1 | tail -1)"
  done
done
