#!/bin/bash
# usage: tools/vbench.sh WL V1 V2 ...  (V = variant name under variants/, or "main" for the in-tree build)
# one short bench line per variant -> gpurun_out/vbench.txt
wl=$1; shift
for v in "$@"; do
  lib=""; [ "$v" != "main" ] && lib="TRMCR_LIB=variants/libtrmcr_$v.so"
  env $lib $VENV timeout 300 python bench.py --workload $wl --no-cpu-baseline --secondary none --steps ${STEPS:-20} > gpurun_out/vb_$v.json 2> gpurun_out/vb_$v.err
  python - "$v" "$wl" <<'PY' >> gpurun_out/vbench.txt
import json, sys
try:
    d = json.loads(open(f"gpurun_out/vb_{sys.argv[1]}.json").read())
    kp = {k: v for k, v in d["roofline"]["kernel_ms_probe"].items() if v > 0.0075}
    print(sys.argv[1], sys.argv[2], f"{d['ms_per_step']:.4f}ms", kp)
except Exception as e:
    print(sys.argv[1], sys.argv[2], "FAILED", e)
PY
done
