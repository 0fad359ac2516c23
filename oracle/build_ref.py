"""Install the UNMODIFIED reference package into ``oracle/_ref/`` — TEST INFRASTRUCTURE ONLY.

    python oracle/build_ref.py          # in the build container (needs /root/reference)

The reference (``/root/reference/pkg``, the pure-Python ``nnmg`` package) is
pip-installed offline from a scratch copy (``/root/reference`` is read-only and
setuptools writes build files next to the sources) with ``--target oracle/_ref``.
``oracle/_ref/`` is git-ignored (no reference source enters the history) but
not gpurun-ignored, so the installed package travels to the GPU box like the
built ``.so``.  It is used as

* the checker of the drop-in test (``tests/test_gpu_dropin_reference.py``): the
  GPU operator / transfer / smoother / coarse-solver objects are plugged into
  the reference's own ``nnmg.multigrid.MultigridHierarchy`` over the reference's
  own ``FESpace`` objects and compared with the all-NumPy reference hierarchy;
* ``bench.py --impl reference`` and the ``cpu_baseline`` leg (``kind:
  "reference"``): the reference's own V-cycle timed on the host cores.

The product package never imports it.  ``ref_path()`` returns the directory to
put on ``sys.path`` (or None when the install is absent, e.g. in a checkout
that never ran ``build()`` where /root/reference exists).
"""

from __future__ import annotations

import os
import shutil
import subprocess
import sys
import tempfile

HERE = os.path.dirname(os.path.abspath(__file__))
DEST = os.path.join(HERE, "_ref")
SRC = "/root/reference/pkg"


def ref_path():
    return DEST if os.path.exists(os.path.join(DEST, "nnmg", "multigrid.py")) else None


def import_reference():
    """The reference ``nnmg`` package from oracle/_ref, or None."""
    p = ref_path()
    if p is None:
        return None
    if p not in sys.path:
        sys.path.insert(0, p)
    import nnmg  # noqa: F401

    return nnmg


def build(force=False):
    if not os.path.isdir(SRC):
        return ref_path()
    if ref_path() is not None and not force:
        return DEST
    tmp = tempfile.mkdtemp(prefix="nnmg_ref_")
    try:
        work = os.path.join(tmp, "pkg")
        shutil.copytree(SRC, work)
        if os.path.isdir(DEST):
            shutil.rmtree(DEST)
        cmd = [sys.executable, "-m", "pip", "install", "--no-index", "--no-build-isolation", "--no-deps",
               "--find-links", "/opt/wheelhouse", "--target", DEST, work]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError("reference install failed:\n" + r.stdout[-2000:] + r.stderr[-2000:])
    finally:
        shutil.rmtree(tmp, ignore_errors=True)
    return ref_path()


if __name__ == "__main__":
    print(build(force="--force" in sys.argv))
