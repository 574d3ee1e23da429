#!/bin/bash
# GMM + PBAS concurrency: K1 capped by dynamic shared memory so PBAS blocks fit beside it.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
export RGBDSEG_B200_AUTOBUILD=0
for lib in "" tuning/lib_gmmpad*.so; do
  tag=${lib:-default}; tag=$(basename "$tag" .so)
  for prio in 0 1; do
  RGBDSEG_B200_LIB=${lib:+$PWD/$lib} timeout 300 python bench.py --no-e2e --no-cpu-baseline --no-verify --steps 50 --stream-priority $prio \
    > gpurun_out/ov.json 2>/dev/null
  echo "$tag prio=$prio $(python -c "import json;d=json.load(open('gpurun_out/ov.json'));print(round(d['ms_per_step'],4), {k:round(v['ms_per_step'],4) for k,v in d['per_algo'].items()})")"
  done
done
