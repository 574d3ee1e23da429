#!/bin/bash
# Strip-K2 sweep at T = t_lower (8 x 1080p, K2 pinned to the "many updates" variant):
# ms per frame for the default library and tuning/lib_*.so variants, L2 prefetch distances.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
export RGBDSEG_B200_AUTOBUILD=0
for lib in "" tuning/lib_*.so; do
  tag=${lib:-default}; tag=$(basename "$tag" .so)
  for pf in 0; do
    echo "$tag pf=$pf $(RGBDSEG_B200_LIB=${lib:+$PWD/$lib} timeout 300 python scripts/micro/pbas_t2_time.py 2 2>&1 | tail -1)"
  done
done
