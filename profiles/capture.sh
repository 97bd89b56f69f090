#!/bin/bash
# ncu captures behind profiles/ (run under gpurun on one B200; never a multi-rank command).
# $1 = round tag (e.g. r1). Outputs land in gpurun_out/ and are summarised by profiles/summarize.py.
set -u
R=${1:-r1}
for c in rbm mlp mnist_cnn cifar_cnn; do
  ncu --metrics gpu__time_duration.sum --clock-control none --csv \
      --log-file gpurun_out/${R}_launches_${c}.csv \
      python bench.py --profile-only --config $c --steps 3 --warmup 2 > /dev/null 2>&1
done
# one full step of the headline workload (RBM CD-1: 4 GEMM launches), full metric set
ncu --set full --clock-control none --import-source on -k regex:gemm_tc -s 8 -c 4 \
    -o gpurun_out/${R}_rbm_full python bench.py --profile-only --config rbm --steps 3 --warmup 2 > /dev/null 2>&1
# the conv kernels of the CIFAR step (fwd x2, dgrad, wgrad x2)
ncu --set full --clock-control none --import-source on -k regex:conv_tc -s 6 -c 6 \
    -o gpurun_out/${R}_cifar_conv_full python bench.py --profile-only --config cifar_cnn --steps 2 --warmup 1 > /dev/null 2>&1
ls -la gpurun_out
