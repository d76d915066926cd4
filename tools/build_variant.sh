#!/bin/bash
# Build a library variant with extra nvcc defines into variants/<name>.so (A/B runs via LG_LIB_PATH):
#   bash tools/build_variant.sh dnreg96 -DLG_DUNGEON_S_NREG=96
name=$1; shift
mkdir -p variants
python - "$name" "$@" <<'PY'
import subprocess, sys, os
sys.path.insert(0, os.getcwd())
from paper_2408_12525_b200 import build as b
name, extra = sys.argv[1], sys.argv[2:]
cmd = [b.nvcc(), *b.NVCC_FLAGS, *extra, "-I", os.path.join(b.ROOT, "include"), b.SRC, b.HOST_SRC,
       "-Xcompiler", "-pthread", "-o", f"variants/{name}.so"]
r = subprocess.run(cmd, capture_output=True, text=True)
open(f"variants/{name}.ptxas.log", "w").write(r.stdout + r.stderr)
print(name, "rc", r.returncode)
PY
