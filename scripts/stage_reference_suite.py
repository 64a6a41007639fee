"""Copy the reference's test files into tests/reference_suite/_staged/
(git-ignored, not gpurun-ignored) so the GPU box can run them against this
package under the name ``hjls`` (tests/reference_suite/conftest.py).
Needs /root/reference (this container); the copies are never committed."""
import glob
import os
import shutil
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = "/root/reference/pkg/tests"
DST = os.path.join(ROOT, "tests", "reference_suite", "_staged")

if not os.path.isdir(SRC):
    sys.exit(f"{SRC} not found: stage the suite where the reference is present")
os.makedirs(DST, exist_ok=True)
n = 0
for f in sorted(glob.glob(os.path.join(SRC, "*.py"))):
    shutil.copy(f, DST)
    n += 1
open(os.path.join(DST, "__init__.py"), "a").close()
print(f"staged {n} reference test files into {DST}")
