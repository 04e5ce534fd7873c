#!/bin/bash
# Round evidence on one B200: bench lines (C3 default with CPU baseline, C4, C5),
# the reference (oracle) arm, smoke(), the ncu launch list of the default bench
# command and --set full captures of the dominant kernels.  Output: gpurun_out/ev/
set -x
mkdir -p gpurun_out/ev
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/ev/smoke.log 2>&1
python bench.py > gpurun_out/ev/bench_c3.json 2> gpurun_out/ev/bench_c3.err
python bench.py --workload c4 > gpurun_out/ev/bench_c4.json 2> gpurun_out/ev/bench_c4.err
python bench.py --workload c5 --steps 300 > gpurun_out/ev/bench_c5.json 2> gpurun_out/ev/bench_c5.err
python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/ev/ref_c3.json 2> gpurun_out/ev/ref_c3.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 300 --csv --log-file gpurun_out/ev/c3_launches.csv \
    python bench.py --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/ev/ncu_launch.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:thermal_warp_kernel -s 2 -c 1 \
    -o gpurun_out/ev/c3_thermal python tools/prof_run.py c3 4 > gpurun_out/ev/ncu_c3.log 2>&1
for k in shock_collide_lock scatter_sorted transport_kernel; do
  ncu --set full --clock-control none --import-source on -k regex:$k -s 2 -c 1 \
      -o gpurun_out/ev/c5_$k python tools/prof_run.py c5 4 > gpurun_out/ev/ncu_c5_$k.log 2>&1
done
ncu --set full --clock-control none --import-source on -k regex:shock_collide_lock -s 2 -c 1 \
    -o gpurun_out/ev/c4_shock_collide_lock python tools/prof_run.py c4 4 > gpurun_out/ev/ncu_c4.log 2>&1
ls -la gpurun_out/ev
# summaries on the box (the copy-back limit is 64 MiB)
for r in gpurun_out/ev/*.ncu-rep; do
  b=${r%.ncu-rep}
  python tools/ncu_summary.py $r > $b.summary.json 2>/dev/null
  ncu -i $r --page source --csv --print-source cuda,sass > $b.src.csv 2>/dev/null && python tools/ncu_hot.py $b.src.csv 40 > $b.hot.txt; rm -f $b.src.csv
done
rm -f gpurun_out/ev/*.ncu-rep   # the copy-back limit is 64 MiB: summaries only
du -sh gpurun_out/ev; ls -la gpurun_out/ev
