#!/bin/bash
# Tile-K2 height sweep: PBAS per-frame cost vs model age (auto K2 variant) for tuning/lib_th*.so.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
export RGBDSEG_B200_AUTOBUILD=0
for lib in "" tuning/lib_th*.so; do
  tag=${lib:-th8}; tag=$(basename "$tag" .so)
  RGBDSEG_B200_LIB=${lib:+$PWD/$lib} timeout 600 python scripts/micro/pbas_age.py > gpurun_out/age_$tag.txt 2>&1
  echo "$tag $(python -c "
import json
rows=[json.loads(l) for l in open('gpurun_out/age_$tag.txt') if l.startswith('{')]
print([(r['frame'], round(r['ms_per_frame'],3)) for r in rows])")"
done
