"""Build the library of a git revision as an A/B variant of the working tree:
python tools/build_base.py [REV] -> paper_2303_15491_b200/libplmss_b200_base.so
(then tools/ab.sh base on the GPU box)."""
import os
import subprocess
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2303_15491_b200 import _build  # noqa: E402

rev = sys.argv[1] if len(sys.argv) > 1 else "HEAD"
tmp = tempfile.mkdtemp(prefix="plmss_base_")
for sub, dst in (("paper_2303_15491_b200/csrc", "csrc"), ("include", "include")):
    os.makedirs(os.path.join(tmp, dst), exist_ok=True)
    names = subprocess.run(["git", "-C", ROOT, "ls-tree", "--name-only", f"{rev}:{sub}"], check=True,
                           capture_output=True, text=True).stdout.split()
    for n in names:
        blob = subprocess.run(["git", "-C", ROOT, "show", f"{rev}:{sub}/{n}"], capture_output=True)
        if blob.returncode == 0:
            with open(os.path.join(tmp, dst, n), "wb") as fh:
                fh.write(blob.stdout)
_build.CSRC = os.path.join(tmp, "csrc")
_build.INCLUDE = os.path.join(tmp, "include")
_build.NVCC_FLAGS = [f for f in _build.NVCC_FLAGS if not f.startswith("-I")] + ["-I" + _build.INCLUDE,
                                                                                "-I" + _build.CSRC]
print(_build.build_cuda(force=True, variant="base"))
