"""Build an A/B variant of libdsp.so with extra nvcc flags (same sources):
    python scripts/variant.py NAME -DFOO=1 ...  ->  paper_2403_10266_b200/libdsp_NAME.so
Select it at run time with DSP_LIB_OVERRIDE=<path> (experiments only)."""
import os, subprocess, sys, concurrent.futures as cf
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2403_10266_b200 import build as b
name, extra = sys.argv[1], sys.argv[2:]
out_dir = os.path.join(b.ROOT, "build", "variant_" + name)
os.makedirs(out_dir, exist_ok=True)
def comp(src):
    obj = os.path.join(out_dir, src + ".o")
    path = os.path.join(b.CSRC, src)
    cmd = [b.NVCC, *b.ARCH, *b.FLAGS, *extra, "-c", path, "-o", obj]
    if src.endswith(".cpp"):
        cmd = [b.NVCC, *b.FLAGS, *extra, "-x", "c++", "-c", path, "-o", obj]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode:
        raise SystemExit(r.stderr)
    return obj
with cf.ThreadPoolExecutor(8) as ex:
    objs = list(ex.map(comp, b._sources()))
lib = os.path.join(b.PKG, f"libdsp_{name}.so")
subprocess.run([b.NVCC, *b.ARCH, "-shared", "-o", lib, *objs, "-cudart", "static", "-ldl", "-lpthread"], check=True)
print("built", lib)
