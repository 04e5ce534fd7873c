#!/bin/bash
# usage: tools/build_variant.sh NAME "-DFLAG=.. -DFLAG2=.."  -> variants/libtrmcr_NAME.so (experiments; TRMCR_LIB selects it)
name=$1; shift
cd "$(dirname "$0")/.."
python - "$name" "$@" <<'PY'
import subprocess, sys
sys.path.insert(0, "paper_1009_2768_b200")
import build as b
flags = sys.argv[2].split() if len(sys.argv) > 2 else []
cmd = [b.NVCC, *b.FLAGS, *flags, "-o", f"variants/libtrmcr_{sys.argv[1]}.so", b.SRC, *b.nccl_flags()]
r = subprocess.run(cmd, capture_output=True, text=True)
print(sys.argv[1], r.returncode, r.stderr[-2000:] if r.returncode else "")
PY
