"""Build an A/B variant of libgs.so from a patched copy of csrc/ (experiments only).

    python tools/build_variant.py NAME FILE 'python-expression-old' 'new' [FILE old new ...]

Copies paper_2311_16728_b200/csrc to /tmp/variant_NAME, replaces each `old` (must occur) with
`new` in FILE, compiles with the package's flags into ab/libgs_NAME.so.  Run the variant with
GS_LIB_PATH=ab/libgs_NAME.so (the .so travels to the GPU box with the snapshot).
"""
import os
import shutil
import subprocess
import sys
import concurrent.futures as cf

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2311_16728_b200 import build as B  # noqa: E402

name = sys.argv[1]
src = f"/tmp/variant_{name}"
shutil.rmtree(src, ignore_errors=True)
shutil.copytree(B.CSRC, src)
args = sys.argv[2:]
for k in range(0, len(args), 3):
    f, old, new = args[k:k + 3]
    p = os.path.join(src, f)
    s = open(p).read()
    assert old in s, f"{old!r} not in {f}"
    open(p, "w").write(s.replace(old, new))
os.makedirs(os.path.join(ROOT, "ab"), exist_ok=True)
flags = [x if x != B.CSRC else src for x in B.FLAGS]


def cc(f):
    o = f"{src}/{os.path.basename(f)}.o"
    r = subprocess.run([B.NVCC, *B.ARCH, *flags, "-c", f, "-o", o], capture_output=True, text=True)
    if r.returncode:
        raise SystemExit(r.stderr)
    return o


srcs = sorted(os.path.join(src, f) for f in os.listdir(src) if f.endswith(".cu"))
with cf.ThreadPoolExecutor(8) as ex:
    objs = list(ex.map(cc, srcs))
out = os.path.join(ROOT, "ab", f"libgs_{name}.so")
r = subprocess.run([B.NVCC, *B.ARCH, "-shared", "-o", out, *objs, "-lcudart_static", "-lrt", "-ldl", "-lpthread"],
                   capture_output=True, text=True)
if r.returncode:
    raise SystemExit(r.stderr)
print(out)
