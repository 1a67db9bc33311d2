"""With hetsched importable, the GPU path's exception classes ARE the
reference's (hetsched/errors.py:4-62), so `except SimError` in the reference
CLI (cli.py:297-301) catches them; ConfidenceVector is the reference class.
Runs in a subprocess with /root/reference on sys.path (build container only)."""

import os
import subprocess
import sys

import pytest

from tests.conftest import REFERENCE_SRC, ROOT

pytestmark = pytest.mark.reference

CODE = r"""
import sys
sys.dont_write_bytecode = True
sys.path[:0] = [{root!r}, {ref!r}]
import hetsched.errors as ref_err
import hetsched.router as ref_router
from paper_2603_22206_b200 import errors, _lib
from paper_2603_22206_b200.router import ConfidenceVector, ConstantRouter
assert errors.REFERENCE_CLASSES
for n in ("SimError", "ValidationError", "DuplicateRequest", "UnknownRequest",
          "UnknownStage", "UnknownModel", "AssignmentConflict"):
    assert getattr(errors, n) is getattr(ref_err, n), n
assert ConfidenceVector is ref_router.ConfidenceVector
import hetsched.balancer as ref_bal
from paper_2603_22206_b200.config import Decision
assert Decision is ref_bal.Decision
try:
    _lib.raise_device_error([_lib.CHM_ERR_DUPLICATE_REQUEST, 3, 1, 0], "t")
except ref_err.SimError as exc:
    assert type(exc) is ref_err.DuplicateRequest
else:
    raise AssertionError("not raised")
from hetsched.profiles import ModelProfile, Pool
pool = Pool((ModelProfile("a", 1.0, 1), ModelProfile("b", 2.0, 2)))
cv = ConstantRouter(0.25).score(None, None, pool)
assert isinstance(cv, ref_router.ConfidenceVector) and cv["b"] == 0.25
print("ok")
"""


def test_errors_are_the_reference_classes():
    code = CODE.format(root=ROOT, ref=REFERENCE_SRC)
    env = dict(os.environ, PYTHONDONTWRITEBYTECODE="1")
    out = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, env=env,
                         timeout=120)
    assert out.returncode == 0, out.stderr[-2000:]
    assert out.stdout.strip().endswith("ok")
