#!/bin/bash
# Round-2 evidence on one B200 -> gpurun_out/ev2/: the default bench line (C5 +
# C3 secondary, CPU baseline), the oracle arm, the ncu launch list of the bench
# command, and --set full captures (summary, hot lines, SASS mix) of the
# dominant kernels.
set -x
mkdir -p gpurun_out/ev2
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/ev2/smoke.log 2>&1
python bench.py > gpurun_out/ev2/bench.json 2> gpurun_out/ev2/bench.err
python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/ev2/ref.json 2> gpurun_out/ev2/ref.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/ev2/c5_launches.csv \
    python bench.py --steps 3 --warmup 3 --no-cpu-baseline --secondary none > gpurun_out/ev2/ncu_launch.log 2>&1
for spec in "shock_collide_lock c5" "scatter_sorted c5" "transport_kernel c5" "thermal_warp_kernel c3"; do
  set -- $spec
  tools/ncu_one.sh $1 $2 ${2}_$1 4
  mv gpurun_out/ncu_${2}_$1.* gpurun_out/ev2/ 2>/dev/null
done
ls -la gpurun_out/ev2
