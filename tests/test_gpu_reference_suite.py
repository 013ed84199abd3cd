"""The reference's own test suite, unmodified, against the drop-in (GPU).

`trackforge` is aliased to this package's hot-path modules (tests/refalias.py),
so the reference's unit, property, oracle, sequence and acceptance tests
(pkg/tests/test_{core,postproc,motion,assoc,tracker,acceptance}.py, SURVEY.md
section 4) call the GPU implementation; the pipeline / CLI / metrics tests run
the reference's own runtime around the GPU tracker.

The suite is the reference's source and is not part of this repository: it
is copied next to the pip-installed reference under the git-ignored
baseline/_ref (tools/stage_reference.sh) and skipped where absent.
"""

import os
import re
import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu

ROOT = Path(__file__).resolve().parents[1]
SUITE = ROOT / "baseline" / "_ref" / "reference_tests"
HOT = ["test_core.py", "test_postproc.py", "test_motion.py", "test_assoc.py", "test_tracker.py",
       "test_acceptance.py"]
REST = ["test_moteval.py", "test_pipeline.py", "test_detgen.py", "test_cli.py"]


def _run(files, tmp_path):
    env = dict(os.environ)
    env["PYTHONPATH"] = os.pathsep.join([str(ROOT / "tests"), str(ROOT), env.get("PYTHONPATH", "")])
    cmd = [sys.executable, "-m", "pytest", "-p", "refalias", "-p", "no:cacheprovider", "-q", "-x",
           "--rootdir", str(SUITE), *[str(SUITE / f) for f in files]]
    res = subprocess.run(cmd, cwd=tmp_path, env=env, capture_output=True, text=True, timeout=1800)
    tail = res.stdout[-3000:] + res.stderr[-2000:]
    m = re.search(r"(\d+) passed", res.stdout)
    return res.returncode, int(m.group(1)) if m else 0, tail


@pytest.mark.skipif(not SUITE.exists(), reason="reference suite not staged (baseline/_ref/reference_tests)")
def test_reference_hot_path_tests_pass_on_the_drop_in(tmp_path):
    rc, passed, tail = _run(HOT, tmp_path)
    print(tail)
    assert rc == 0, tail
    assert passed >= 100


@pytest.mark.skipif(not SUITE.exists(), reason="reference suite not staged (baseline/_ref/reference_tests)")
def test_reference_runtime_tests_pass_around_the_drop_in(tmp_path):
    rc, passed, tail = _run(REST, tmp_path)
    print(tail)
    assert rc == 0, tail
