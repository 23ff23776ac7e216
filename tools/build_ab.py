"""Build an A/B variant of the library: python tools/build_ab.py NAME "EXTRA NVCC FLAGS" file1.cu [file2.cu ...]
recompiles only the listed sources with the extra flags (the other objects come
from the in-tree build) and links _ab/NAME.so; run with MF_LIB_PATH=_ab/NAME.so."""
import os
import subprocess
import sys

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
from paper_1912_13282_b200 import build as b  # noqa: E402

name, extra, files = sys.argv[1], sys.argv[2].split(), sys.argv[3:]
b.build()
out = os.path.join(REPO, "_ab")
os.makedirs(os.path.join(out, name), exist_ok=True)
flags = b.ARCH + ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "--expt-relaxed-constexpr",
                  "-I", os.path.join(REPO, "include"), "-Xptxas", "-warn-spills"] + extra
objs, procs = [], []
for s in b.SOURCES:
    if s in files:
        o = os.path.join(out, name, s + ".o")
        procs.append(subprocess.Popen([b.nvcc(), *flags, "-c", os.path.join(b.CSRC, s), "-o", o]))
    else:
        o = os.path.join(b.HERE, "_build", s + ".o")
    objs.append(o)
if any(p.wait() for p in procs):
    sys.exit("nvcc failed")
lib = os.path.join(out, name + ".so")
subprocess.run([b.nvcc(), *b.ARCH, "-shared", "-o", lib, *objs], check=True)
print(lib)
