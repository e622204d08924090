"""Checked-build runs (the stand-in for compute-sanitizer, which is closed on the GPU pool; see
profiles/r02_sanitizers.md): the library built with -DBSF_CHECKED poisons each kernel's shared memory with NaN
before use, and every output buffer is NaN-filled inside sentinel guard zones.  Every assembly kernel (core,
band, corners, tile, generic, G3-FULL, slabs) must then (1) leave the guards intact (no global write outside
its outputs), (2) write every output entry with a finite value (no output skipped, no read of shared memory it
did not write in this launch), (3) give bit-identical results on repeated calls (no race between warps), and
(4) match the oracle within the north star's 1e-10."""
import json
import os
import subprocess
import sys
import tempfile

import pytest

from parity import TOL

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_checked_build_all_kernels():
    from paper_2506_18867_b200 import build as b
    lib = b.build_checked()
    env = dict(os.environ, BSF_LIB_PATH=lib, BSF_REBUILD="0")
    with tempfile.TemporaryDirectory() as td:
        out = os.path.join(td, "rep.json")
        r = subprocess.run([sys.executable, os.path.join(ROOT, "tests", "_checked_worker.py"), out], env=env,
                           capture_output=True, text=True, timeout=1200, cwd=ROOT)
        assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
        reps = json.load(open(out))
    assert len(reps) == 9
    for rep in reps:
        assert rep["guards_intact"] and rep["finite"] and rep["deterministic"], rep
        assert rep["rel_E"] <= TOL and rep["rel_g"] <= TOL and rep["rel_H"] <= TOL, rep
