"""The reference's own test suite (/root/reference/pkg/tests, 147 tests) run against THIS package.

A shim package named `tpshift` (written to a temp dir) re-exports paper_2605_23945_b200 and maps
every tpshift submodule (cluster, config, controller, engine, errors, latency, reshard,
switchcost, workload) to this package's module of the same name; only the reference's CLI
front-end (tpshift/cli.py, out of scope per SURVEY 8) is loaded from the reference itself, on top
of this package's modules. The suite must pass unchanged: a tpshift user switching imports to
this package finds every name, value and behaviour the reference's tests pin (decisions, plans,
predictor, switch costs, reports, presets). Container only (reads /root/reference).
"""

import os
import shutil
import subprocess
import sys

import pytest

pytestmark = pytest.mark.reference

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = "/root/reference/pkg"

SHIM = '''import importlib.util as _u
import sys
import paper_2605_23945_b200 as _p
from paper_2605_23945_b200 import *  # noqa: F401,F403
for _m in ("cluster", "config", "controller", "engine", "errors", "latency", "reshard", "switchcost", "workload"):
    _mod = __import__("paper_2605_23945_b200." + _m, fromlist=["x"])
    sys.modules["tpshift." + _m] = _mod
    globals()[_m] = _mod
for _n in dir(_p):
    if not _n.startswith("__"):
        globals().setdefault(_n, getattr(_p, _n))
_spec = _u.spec_from_file_location("tpshift.cli", "%s/src/tpshift/cli.py")
cli = _u.module_from_spec(_spec)
sys.modules["tpshift.cli"] = cli
_spec.loader.exec_module(cli)
''' % REF


def test_reference_test_suite_passes_against_this_package(tmp_path):
    shim = tmp_path / "shim" / "tpshift"
    shim.mkdir(parents=True)
    (shim / "__init__.py").write_text(SHIM)
    suite = tmp_path / "suite"
    shutil.copytree(os.path.join(REF, "tests"), suite)
    env = dict(os.environ, PYTHONPATH=os.pathsep.join([str(tmp_path / "shim"), ROOT]))
    which = subprocess.run([sys.executable, "-c", "import tpshift; print(tpshift.evaluate.__module__)"],
                           cwd=suite, env=env, capture_output=True, text=True, check=True).stdout.strip()
    assert which == "paper_2605_23945_b200.controller"
    res = subprocess.run([sys.executable, "-m", "pytest", "-q", "-p", "no:cacheprovider", str(suite)],
                         cwd=suite, env=env, capture_output=True, text=True, timeout=900)
    tail = res.stdout.strip().splitlines()[-1]
    assert res.returncode == 0, res.stdout[-3000:]
    assert "147 passed" in tail, tail
