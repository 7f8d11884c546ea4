"""Install the UNMODIFIED reference package (volkrig) into the git-ignored
``baseline/_ref`` so ``bench.py --impl reference`` (and the bench line's
``cpu_baseline``) can time the reference's own ``fit_variogram`` +
``fill_missing`` on the GPU box's host cores.

The install is the one offline ``pip install --target`` the task allows:
no index, no build isolation, ``--no-deps`` (numpy / scipy / Pillow come
from the image).  ``/root/reference`` is read-only, so the package is built
from a copy under /tmp.  ``baseline/_ref`` travels to the GPU box with the
gpurun snapshot (git-ignored, not gpurun-ignored); nothing at run time reads
``/root/reference``.

Run: ``python tools/vendor_ref.py`` (``build()`` calls it when the reference
is mounted).  Exit 0 and a one-line status either way.
"""

from __future__ import annotations

import os
import shutil
import subprocess
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = "/root/reference/pkg"
DEST = os.path.join(ROOT, "baseline", "_ref")


def installed() -> bool:
    return os.path.isfile(os.path.join(DEST, "volkrig", "kriging.py"))


def vendor(force: bool = False) -> str:
    if installed() and not force:
        return f"reference already installed in {DEST}"
    if not os.path.isdir(SRC):
        return f"reference not mounted ({SRC}); {DEST} left as is"
    tmp = tempfile.mkdtemp(prefix="volkrig_src_")
    try:
        work = os.path.join(tmp, "pkg")
        shutil.copytree(SRC, work, ignore=shutil.ignore_patterns("__pycache__", "*.pyc", "build",
                                                                  "*.egg-info"))
        if os.path.isdir(DEST):
            shutil.rmtree(DEST)
        os.makedirs(DEST, exist_ok=True)
        cmd = [sys.executable, "-m", "pip", "install", "--no-index", "--no-build-isolation",
               "--no-deps", "--find-links", "/opt/wheelhouse", "--target", DEST, "--quiet", work]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0 or not installed():
            return f"pip install of the reference failed ({r.returncode}): {r.stderr.strip()[-300:]}"
        return f"reference installed in {DEST}"
    finally:
        shutil.rmtree(tmp, ignore_errors=True)


if __name__ == "__main__":
    print(vendor(force="--force" in sys.argv))
