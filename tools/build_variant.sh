#!/bin/bash
# build the library with extra nvcc flags (e.g. -DCNRX_BLK_RELU_WARPS=5) into abtest/lib_<name>.so
# usage: tools/build_variant.sh name "-DFOO=1 -DBAR=2"
set -e
cd "$(dirname "$0")/.."
name=$1; shift
D=/tmp/cnrx_variant_$name
rm -rf $D && mkdir -p $D
cp -r paper_2510_12739_b200/csrc $D/csrc
python - "$name" "$*" <<'PY'
import os, sys, subprocess
sys.path.insert(0, ".")
from paper_2510_12739_b200 import build as B
name, extra = sys.argv[1], sys.argv[2]
D = f"/tmp/cnrx_variant_{name}"
objs = []
def comp(src):
    obj = os.path.join(D, os.path.splitext(src)[0] + ".o")
    cmd = [B.nvcc()] + B.flags() + extra.split() + B.SOURCE_FLAGS.get(src, []) + ["-c", os.path.join(B.CSRC, src), "-o", obj]
    subprocess.run(cmd, check=True)
    return obj
import concurrent.futures as cf
with cf.ThreadPoolExecutor(8) as ex:
    objs = list(ex.map(comp, B.SOURCES))
os.makedirs("abtest", exist_ok=True)
subprocess.run([B.nvcc(), "-shared", "-o", f"abtest/lib_{name}.so"] + objs + B.ARCH + ["-cudart", "static", "-ccbin", B.host_cxx(), "-ldl", "-lpthread"], check=True)
print(f"abtest/lib_{name}.so")
PY
