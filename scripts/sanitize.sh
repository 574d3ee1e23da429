#!/bin/bash
# compute-sanitizer memcheck / racecheck / synccheck over small GPU parity cases
# (every kernel: K1 plain + EVAL, K2 both intent modes + EVAL, K3 map + list,
# pack, median, rng, fast divide self-test, peer-memory halo push/pull; round 2:
# strip K2 with cp.async staging, fused cooperative K2+K3, staged host paths).
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out/sanitizer
CASES='golden or ragged or row_bands_on_one_gpu or median or pack or confusion or rng or deferred or list_handle or fast_divide or process_sequence or extreme or k2_variants or tile_variant or submit or mixed_input or least_fit or prefilter'
for tool in memcheck racecheck synccheck; do
  timeout 1500 compute-sanitizer --tool $tool --target-processes all --error-exitcode 9 \
    python -m pytest tests/test_gpu_parity.py tests/test_gpu_bands.py tests/test_gpu_plugin.py -m gpu -q -x \
    -k "$CASES or local_peer_links or plugin" -p no:cacheprovider \
    > gpurun_out/sanitizer/$tool.log 2>&1
  echo "$tool rc=$? $(grep -E 'ERROR SUMMARY|passed|failed' gpurun_out/sanitizer/$tool.log | tail -3 | tr '\n' ' ')"
done
