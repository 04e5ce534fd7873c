#!/bin/bash
# usage: tools/bsum.sh "ENV=.. ENV2=.." c5 c4 ...   -> appends one summary line per run to gpurun_out/bsum.txt
envs="$1"; shift
mkdir -p gpurun_out
for w in "$@"; do
  env $envs python bench.py --workload $w --steps ${STEPS:-200} --no-cpu-baseline > gpurun_out/b_$w.json 2>gpurun_out/b_$w.err
  python - "$envs" "$w" << 'PY' >> gpurun_out/bsum.txt
import json, sys
try:
    d = json.loads(open(f"gpurun_out/b_{sys.argv[2]}.json").read())
    kp = {k: v for k, v in d["roofline"]["kernel_ms_probe"].items() if v > 0.0075}
    print(sys.argv[1] or "-", sys.argv[2], f"{d['value']/1e9:.2f}G/s", f"{d['ms_per_step']:.4f}ms", d["roofline"]["kernel"], d["roofline"]["frac"], kp)
except Exception as e:
    print(sys.argv[1], sys.argv[2], "FAILED", e)
PY
done
