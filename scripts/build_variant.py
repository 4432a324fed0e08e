"""Build a variant of the library with extra -D flags (A/B experiments):
python scripts/build_variant.py NAME -DFOO=1 ...  ->  scripts/_var/NAME.so,
loaded with EPC_LIB=scripts/_var/NAME.so."""
import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

sys.path.insert(0, __file__.rsplit("/scripts/", 1)[0])
from paper_1607_00531_b200 import build as B  # noqa: E402

name, defs = sys.argv[1], sys.argv[2:]
out = os.path.join(os.path.dirname(os.path.abspath(__file__)), "_var")
os.makedirs(out, exist_ok=True)


def cc(src):
    o = os.path.join(out, f"{name}_{os.path.splitext(src)[0]}.o")
    flags = [f for f in B.FLAGS if not (src in B.FMAD_ON and f == "-fmad=false")]
    if src in B.FMAD_ON:
        flags.append("-fmad=true")
    cmd = [B.NVCC, *B.ARCH, *flags, *defs, "-c", os.path.join(B.CSRC, src), "-o", o]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode:
        raise SystemExit(r.stderr)
    return o


with ThreadPoolExecutor(len(B.SOURCES)) as ex:
    objs = list(ex.map(cc, B.SOURCES))
lib = os.path.join(out, f"{name}.so")
subprocess.run([B.NVCC, *B.ARCH, "-shared", "-o", lib, *objs, *B.LIBS], check=True)
for o in objs:  # keep only the library (the snapshot travels to the GPU box)
    os.remove(o)
print(lib)
