"""Build libkaczmarz_b200_ab.so from the current sources with some csrc files replaced (same-box A/B):

    python tools/build_ab.py csrc/kz_solve_wide.cuh=/tmp/old_wide.cuh [...]
then run the same command with KZ_LIB_VARIANT=ab (A) and without (B) in one gpurun call
(--name=X as the first argument builds libkaczmarz_b200_X.so for a third arm, KZ_LIB_VARIANT=X;
-DNAME=VALUE arguments are passed to nvcc for that arm).
"""
import os
import shutil
import subprocess
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2501_10689_b200 import build as B  # noqa: E402

tmp = tempfile.mkdtemp()
src = os.path.join(tmp, "pkg", "csrc")  # keeps csrc/../../include valid
shutil.copytree(B.CSRC, src)
shutil.copytree(os.path.join(ROOT, "include"), os.path.join(tmp, "include"))
name = "ab"
args = sys.argv[1:]
if args and args[0].startswith("--name="):
    name = args.pop(0).split("=", 1)[1]
defs = [x for x in args if x.startswith("-D")]  # extra preprocessor definitions for this arm
args = [x for x in args if not x.startswith("-D")]
for arg in args:
    rel, path = arg.split("=", 1)
    shutil.copy(path, os.path.join(tmp, "pkg", rel))
out = B.lib_path(name)
cmd = [B._nvcc(), *B.NVCC_FLAGS, *defs, "-I", os.path.join(ROOT, "include"), *[os.path.join(src, s) for s in B.SOURCES],
       "-o", out]
res = subprocess.run(cmd, capture_output=True, text=True)
open(out + ".log", "w").write(res.stderr)
if res.returncode:
    sys.stderr.write(res.stderr[-4000:])
    sys.exit(1)
print(out)
