#!/bin/bash
# Build a variant of libtgb.so with extra nvcc -D flags into build/libtgb_<name>.so
# (same-box A/B with tools/lib_ab.sh; the in-tree library is left untouched).
#   tools/build_variant.sh <name> [-DFLAG ...]
set -e
name=$1; shift
python - "$name" "$@" <<'PY'
import subprocess, sys
sys.path.insert(0, ".")
from paper_1705_07878_b200 import build as b
name, flags = sys.argv[1], sys.argv[2:]
_, nccl_lib = b.nccl_dirs()
out = f"build/libtgb_{name}.so"
cmd = [b.NVCC, *b.nvcc_flags(), *flags, "-shared", "-o", out, *b.SOURCES, "-L" + nccl_lib,
       "-l:libnccl.so.2", "-Xlinker", "-rpath=" + nccl_lib, "-lcudart"]
subprocess.run(cmd, check=True)
print(out)
PY
