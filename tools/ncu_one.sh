#!/bin/bash
# ncu --set full of one kernel launch, exported as text next to gpurun_out/ (the .ncu-rep stays in /tmp).
# Usage: tools/ncu_one.sh TAG KERNEL_REGEX command...    (run on the GPU box)
set -u
tag=$1; kre=$2; shift 2
mkdir -p gpurun_out
timeout 300 ncu -f --set full --import-source on --clock-control none -k "regex:${kre}" --launch-skip ${NCU_SKIP:-1} -c 1 \
  -o /tmp/ncu_$tag "$@" > gpurun_out/ncu_$tag.log 2>&1
ncu -i /tmp/ncu_$tag.ncu-rep --page details > gpurun_out/$tag.details.txt 2>&1
ncu -i /tmp/ncu_$tag.ncu-rep --page raw --csv > gpurun_out/$tag.raw.csv 2>&1
ncu -i /tmp/ncu_$tag.ncu-rep --page source --csv --print-source sass > gpurun_out/$tag.sass.csv 2>&1
