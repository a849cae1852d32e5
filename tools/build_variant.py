"""Build an experimental variant of the library with extra nvcc flags (A/B experiments):
python tools/build_variant.py OUT.so -DFLAG=V ..."""
import os
import subprocess
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2408_14302_b200 import build as B  # noqa: E402

out, extra = os.path.abspath(sys.argv[1]), sys.argv[2:]
objdir = out + ".objs"
os.makedirs(objdir, exist_ok=True)
cflags = [f for f in B.FLAGS if f != "-shared"] + extra
procs = []
for src in B.sources():
    obj = os.path.join(objdir, os.path.basename(src)[:-3] + ".o")
    procs.append((obj, subprocess.Popen([B.NVCC, *cflags, "-c", "-o", obj, src], stdout=subprocess.PIPE,
                                        stderr=subprocess.PIPE, text=True)))
log = ""
for obj, pr in procs:
    o, e = pr.communicate()
    log += e
    if pr.returncode:
        sys.exit(o + e)
subprocess.run([B.NVCC, "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o", out, *[o for o, _ in procs]],
               check=True)
open(out + ".ptxas.log", "w").write(log)
print(out)
