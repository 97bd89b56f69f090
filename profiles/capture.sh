#!/bin/bash
# ncu captures behind profiles/ (run under gpurun on one B200; never a multi-rank command).
# $1 = round tag (e.g. r1). Outputs land in gpurun_out/ and are summarised by profiles/summarize.py.
set -u
R=${1:-r1}
for c in rbm mlp mnist_cnn cifar_cnn imagenet_cnn crbm; do
  ncu --metrics gpu__time_duration.sum --clock-control none --csv \
      --log-file gpurun_out/${R}_launches_${c}.csv \
      python bench.py --profile-only --config $c --steps 1 --warmup 1 > /dev/null 2>&1
done
# one step of the headline workload: the fused CD-1 kernel, and the 4-GEMM split path it replaced
ncu --set full --clock-control none --import-source on -k regex:rbm_cd1 -s 1 -c 1 \
    -o gpurun_out/${R}_rbm_full python bench.py --profile-only --config rbm --steps 1 --warmup 1 > /dev/null 2>&1
B2N_RBM_FUSED=0 ncu --set full --clock-control none --import-source on -k regex:gemm_tc -s 4 -c 4 \
    -o gpurun_out/${R}_rbm_split_full python bench.py --profile-only --config rbm --steps 1 --warmup 1 > /dev/null 2>&1
# the one-launch convolutional-RBM step and its split tensor-core path
ncu --set full --clock-control none --import-source on -k regex:crbm_cd1_fused -s 2 -c 1 \
    -o gpurun_out/${R}_crbm_full python bench.py --profile-only --config crbm --steps 1 --warmup 2 > /dev/null 2>&1
B2N_CRBM_FUSED=0 ncu --set full --clock-control none --import-source on -k regex:"conv_tc_kernel|crbm_update" -s 10 -c 5 \
    -o gpurun_out/${R}_crbm_split_full python bench.py --profile-only --config crbm --steps 1 --warmup 2 > /dev/null 2>&1
# the halo-tile conv kernels of one ImageNet-shape step (5 fwd, 4 dgrad, 5 wgrad)
ncu --set full --clock-control none --import-source on -k regex:"convt_(mma|wgrad)_kernel" -c 14 \
    -o gpurun_out/${R}_imagenet_conv_full python bench.py --profile-only --config imagenet_cnn --steps 1 --warmup 0 > /dev/null 2>&1
ls -la gpurun_out
