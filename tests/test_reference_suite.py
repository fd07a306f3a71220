"""The reference's own unit tests, run against this package (the drop-in check).

``fp8sta`` and its submodules are aliased to ``paper_2506_04648_b200`` inside a
subprocess pytest run of the reference's test files (read from
/root/reference, so these run in the build container only; the GPU box has no
reference tree).  Host-side files only -- grid, sparsity, schedule: the
quantiser / codec / attention tests need a GPU and are covered by the golden
vectors the reference generated (tests/golden, test_gpu_*.py).  The
reference's conftest is skipped (--noconftest): it imports fp8sta.experiment,
the out-of-scope experiment runner, for fixtures these files do not use.
"""

import os
import re
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF_TESTS = "/root/reference/pkg/tests"

ALIAS = '''import importlib
import sys

import paper_2506_04648_b200 as pkg

sys.modules["fp8sta"] = pkg
for sub in ("grid", "sparsity", "schedule", "quantize", "fp8", "attention", "metrics"):
    sys.modules["fp8sta." + sub] = importlib.import_module("paper_2506_04648_b200." + sub)
'''


@pytest.mark.skipif(not os.path.isdir(REF_TESTS), reason="reference tree not present")
@pytest.mark.parametrize("name,count", [("test_grid.py", 11), ("test_sparsity.py", 20), ("test_schedule.py", 11)])
def test_reference_unit_tests_pass_against_package(name, count, tmp_path):
    (tmp_path / "fp8sta_alias.py").write_text(ALIAS)
    env = dict(os.environ, PYTHONDONTWRITEBYTECODE="1", PYTHONPATH=f"{tmp_path}{os.pathsep}{ROOT}")
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-p", "fp8sta_alias", "--noconftest", "-p",
                        "no:cacheprovider", os.path.join(REF_TESTS, name)], cwd=tmp_path, env=env,
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]
    m = re.search(r"(\d+) passed", r.stdout)
    assert m and int(m.group(1)) == count, r.stdout[-500:]
