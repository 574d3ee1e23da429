#!/bin/bash
# Multi-rank bench logic on ONE GPU (gloo plumbing, every rank on cuda:0):
# config4 stream digests must not depend on the rank count; config5 row
# bands must be bit-equal to the one-band run.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
export RGBDSEG_B200_AUTOBUILD=0
A="--steps 10 --warmup 3 --no-e2e --no-cpu-baseline"
timeout 300 python bench.py $A > gpurun_out/mr_c4_n1.json 2>gpurun_out/mr_c4_n1.err
RGBDSEG_BENCH_SHARED_GPU=1 timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 \
  --master-addr 127.0.0.1 --master-port 29511 bench.py $A --streams 4 > gpurun_out/mr_c4_n2.json 2>gpurun_out/mr_c4_n2.err
timeout 300 python bench.py $A --streams 4 > gpurun_out/mr_c4_n1s4.json 2>>gpurun_out/mr_c4_n1.err
for n in 2 4; do
  RGBDSEG_BENCH_SHARED_GPU=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n \
    --master-addr 127.0.0.1 --master-port 2952$n bench.py --workload config5 --steps 10 --warmup 3 \
    > gpurun_out/mr_c5_n$n.json 2>gpurun_out/mr_c5_n$n.err
done
python - <<'PY'
import json
def L(p):
    try:
        return json.loads(open(p).read().strip().splitlines()[-1])
    except Exception as e:
        return {"error": str(e)}
a, b, c = L("gpurun_out/mr_c4_n1s4.json"), L("gpurun_out/mr_c4_n2.json"), L("gpurun_out/mr_c4_n1.json")
da, db = a.get("stream_digests") or {}, b.get("stream_digests") or {}
print("c4 n1(4 streams) vs n2(2x4): common ids", sorted(set(da) & set(db)),
      "equal:", all(da[k] == db[k] for k in set(da) & set(db)))
dc = c.get("stream_digests") or {}
print("c4 n1(8 streams) vs n2(2x4) ids 0-7 equal:", all(dc.get(k) == db.get(k) for k in db))
for n in (2, 4):
    d = L(f"gpurun_out/mr_c5_n{n}.json")
    print("c5", n, d.get("bit_equal_across_gpus"), d.get("ranks"), d.get("collective_backend"), d.get("error"))
PY
