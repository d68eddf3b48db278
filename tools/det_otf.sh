# determinism of the on-the-fly weight mode with 2, 3 and 4 weight stages (HG_TC_NBS), after
# the release-before-consume fix: 3 repeats x 2 shapes per variant
for nbs in 2; do   # 3 and 4 no longer fit the shared-memory budget
  # (variants built before the GPU call: tools/build_variant.sh nbs$nbs -DHG_TC_NBS=$nbs)
  for cfg in small dense; do
    for r in 1 2 3; do HEGRID_LIB=tmp_libs/lib_nbs$nbs.so HEGRID_TC_PW=0 timeout 120 python tools/det_small.py $cfg | sed "s/^/NBS=$nbs /"; done
  done
done
