#!/bin/bash
# ncu --set full of one kernel (regex $1, skip $2 launches) of a command, summarised into
# gpurun_out/<tag>_{details.txt,raw.csv,sass.csv,cuda.csv} (the .ncu-rep stays in /tmp: too big).
# usage (on the GPU box): tools/ncu_kernel.sh <kernel-regex> <skip> <tag> <cmd...>
set -e
re=$1; skip=$2; tag=$3; shift 3
"$@" > gpurun_out/${tag}_plain.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:$re -s $skip -c 1 -o /tmp/$tag "$@" > gpurun_out/${tag}_ncu.log 2>&1
ncu -i /tmp/$tag.ncu-rep --page details > gpurun_out/${tag}_details.txt
ncu -i /tmp/$tag.ncu-rep --page raw --csv > gpurun_out/${tag}_raw.csv
ncu -i /tmp/$tag.ncu-rep --page source --csv --print-source sass > gpurun_out/${tag}_sass.csv
ncu -i /tmp/$tag.ncu-rep --page source --csv --print-source cuda > gpurun_out/${tag}_cuda.csv || true
