#!/bin/bash
# usage: tools/ncu_one.sh KERNEL_REGEX WORKLOAD TAG [steps]
# one `ncu --set full` capture of the kernel on a few steps of a bench workload;
# summary JSON, hottest source lines and SASS opcode mix into gpurun_out/ncu_TAG.*
k=$1; wl=$2; tag=$3; steps=${4:-4}
mkdir -p gpurun_out
env $NCU_ENV ncu --set full --clock-control none --import-source on -k regex:$k -s 2 -c 1 \
    -o gpurun_out/ncu_$tag python tools/prof_run.py $wl $steps > gpurun_out/ncu_$tag.log 2>&1
r=gpurun_out/ncu_$tag.ncu-rep
python tools/ncu_summary.py $r > gpurun_out/ncu_$tag.summary.json 2>>gpurun_out/ncu_$tag.log
ncu -i $r --page source --csv --print-source cuda,sass > /tmp/ncu_$tag.src.csv 2>/dev/null
python tools/ncu_hot.py /tmp/ncu_$tag.src.csv 60 > gpurun_out/ncu_$tag.hot.txt 2>>gpurun_out/ncu_$tag.log
ncu -i $r --page source --csv --print-source sass > /tmp/ncu_$tag.sass.csv 2>/dev/null
python tools/ncu_sass_mix.py /tmp/ncu_$tag.sass.csv 30 > gpurun_out/ncu_$tag.mix.txt 2>>gpurun_out/ncu_$tag.log
rm -f $r
