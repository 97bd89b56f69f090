#!/usr/bin/env bash
# compute-sanitizer over the kernel tests (race / sync / memory checks of the hand-written
# kernels). Run on a GPU box from the repo root:
#   gpurun -- 'bash tools/sanitize.sh > gpurun_out/sanitize.log 2>&1'
# Each tool runs a small, representative subset (sanitizer replays are 10-100x slower): the fused
# RBM step, the GEMM epilogues, the halo-tile conv fwd/dgrad/wgrad, the CRBM one-launch step, the
# device mt19937 stream. The product kernels use mbarriers / TMA / tcgen05, which racecheck models only
# for shared memory written by threads; a clean report means no thread-level shared-memory hazard.
set -u
cd "$(dirname "$0")/.."
CS=${CS:-/usr/local/cuda/bin/compute-sanitizer}
SEL=${SEL:-"tests/test_gpu_rbm.py::test_cd1_step tests/test_gpu_gemm.py tests/test_gpu_convt_shapes.py tests/test_gpu_crbm.py::test_crbm_cd1_step tests/test_gpu_rng.py tests/test_gpu_mlp.py::test_wide_softmax_rows"}
status=0
for tool in memcheck racecheck synccheck initcheck; do
    echo "=== compute-sanitizer --tool $tool"
    B2N_SANITIZE=1 timeout 1500 "$CS" --tool "$tool" --target-processes all --print-limit 20 --error-exitcode 99 \
        python -m pytest -x -q -m gpu $SEL -p no:cacheprovider 2>&1 | tail -25
    rc=${PIPESTATUS[0]}
    echo "=== $tool exit $rc"
    [ "$rc" -ne 0 ] && status=1
done
exit $status
