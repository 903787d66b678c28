"""A tpshift caller's values cross the drop-in boundary unchanged (CPU, container only).

Scenarios built by the unmodified reference (/root/reference/pkg/src) convert to this
package's types (interop.from_reference) and run to the byte-identical SimReport JSON of
tpshift.run; converting back (interop.to_reference) gives the reference an equal value.
"""

import sys

import pytest

from paper_2605_23945_b200 import engine
from paper_2605_23945_b200.interop import from_reference, to_reference

pytestmark = pytest.mark.reference


@pytest.fixture(scope="module")
def T():
    sys.path.insert(0, "/root/reference/pkg/src")
    import tpshift
    return tpshift


@pytest.mark.parametrize("preset,overrides", [("paper_a40", {}), ("paper_h100", {}),
                                              ("paper_h100", {"global_batch": 384, "l_max": 8192, "initial_tp": 1}),
                                              ("paper_a40", {"mode": "static"})])
def test_reference_scenario_runs_identically_here(T, preset, overrides):
    spec = T.build_scenario(T.load_config(preset), **overrides)
    mine = from_reference(spec)
    assert type(mine).__module__.startswith("paper_2605_23945_b200")
    assert engine.run(mine).to_json() == T.run(spec).to_json()
    back = to_reference(T, mine)
    assert type(back) is type(spec) and back == spec
