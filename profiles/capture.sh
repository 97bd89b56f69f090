#!/bin/bash
# ncu captures behind profiles/ (run under gpurun on one B200; never a multi-rank command).
# $1 = round tag (e.g. r2). Outputs land in gpurun_out/ and are summarised by profiles/summarize.py.
set -u
R=${1:-r2}
# per-kernel launch lists of one step of every config (cold-cache, serialised: shares, not absolutes)
for c in rbm mlp mnist_cnn cifar_cnn imagenet_cnn crbm; do
  ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
      --log-file gpurun_out/${R}_launches_${c}.csv \
      python bench.py --profile-only --config $c --steps 1 --warmup 1 > /dev/null 2>&1
done
# the headline: the fused CD-1 kernel (full set, source-correlated)
ncu --set full --clock-control none --import-source on -k regex:rbm_cd1 -s 1 -c 1 \
    -o gpurun_out/${R}_rbm_full python bench.py --profile-only --config rbm --steps 1 --warmup 1 > /dev/null 2>&1
# the device Bernoulli generator (words + canonical) of one 50,000-draw step
ncu --set full --clock-control none --import-source on -k regex:"mt_(words|canonical)" -s 2 -c 2 \
    -o gpurun_out/${R}_mt_full python tools/diag/rng_time.py > /dev/null 2>&1
# the one-launch convolutional-RBM step
ncu --set full --clock-control none --import-source on -k regex:crbm_cd1_fused -s 2 -c 1 \
    -o gpurun_out/${R}_crbm_full python bench.py --profile-only --config crbm --steps 1 --warmup 2 > /dev/null 2>&1
# the conv kernels of one ImageNet-shaped step: exact forward (convx), tcgen05 dgrad, FFMA wgrad
ncu --set full --clock-control none --import-source on -k regex:"conv(x|t)_(fwd|mma|wgrad)" -c 19 \
    -o gpurun_out/${R}_imagenet_conv_full python bench.py --profile-only --config imagenet_cnn --steps 1 --warmup 0 > /dev/null 2>&1
# the bandwidth kernels north_star names: softmax-xent rows (1000 classes), wgrad reduce + SGD, repack,
# the packed SGD / Adam passes (data-parallel apply and the split optimizer path)
ncu --set full --clock-control none -k regex:"softmax_xent_rows|convt_wgrad_reduce|convt_repack" -c 6 \
    -o gpurun_out/${R}_bw_imagenet python bench.py --profile-only --config imagenet_cnn --steps 1 --warmup 0 > /dev/null 2>&1
ncu --set full --clock-control none -k regex:"sgd_packed|opt_packed" -c 6 \
    -o gpurun_out/${R}_bw_optim python -m pytest -q -m gpu -p no:cacheprovider tests/test_gpu_optim.py tests/test_gpu_dp.py > /dev/null 2>&1
# raw pages exported on the box; large reports dropped (gpurun brings back <= 64 MiB)
for r in gpurun_out/${R}_*.ncu-rep; do
  ncu -i "$r" --page raw --csv > "${r%.ncu-rep}.raw.csv" 2>/dev/null
  if [ $(stat -c %s "$r") -gt 12000000 ]; then rm -f "$r"; fi
done
ls -la gpurun_out
