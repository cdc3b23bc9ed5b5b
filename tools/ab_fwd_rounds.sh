# forward split-rounds threshold A/B (ab/libttb_base.so against ab/libttb_r0.so)
for r in 1 2 3; do for wl in cfg2 cfg3 cfg3p; do
echo "r1 $(TTB_LIB_PATH=ab/libttb_base.so python tools/cfg_kernels.py $wl 2>&1 | tail -1)"
echo "r0 $(TTB_LIB_PATH=ab/libttb_r0.so python tools/cfg_kernels.py $wl 2>&1 | tail -1)"
done; done
