"""Values crossing the drop-in boundary between the reference package `tpshift` and this one.

The decision layer here restates tpshift's dataclasses with the same names and fields
(tpshift/engine.py ScenarioSpec, tpshift/cluster.py ModelSpec / ClusterSpec / ParallelConfig,
tpshift/workload.py Sample / BatchStatus / LengthDistribution, tpshift/latency.py ProfileTable,
tpshift/switchcost.py calibrations, ...), so a value converts field by field by class name:

    spec = from_reference(tpshift.build_scenario(tpshift.load_config("paper_h100")))
    GlobalCoordinator(spec, geometry("qwen2.5-7b"), World.from_env()).run()   # on B200

and back (`to_reference(tpshift, value)`, e.g. to time the unmodified reference on this
package's inputs, bench.py). Non-dataclass values (numbers, strings, numpy arrays) pass through.
"""

from __future__ import annotations

import dataclasses


def _convert(x, ns):
    if dataclasses.is_dataclass(x) and not isinstance(x, type):
        cls = getattr(ns, type(x).__name__)
        return cls(**{f.name: _convert(getattr(x, f.name), ns) for f in dataclasses.fields(x)})
    if isinstance(x, tuple):
        return tuple(_convert(v, ns) for v in x)
    if isinstance(x, list):
        return [_convert(v, ns) for v in x]
    if isinstance(x, dict):
        return {k: _convert(v, ns) for k, v in x.items()}
    return x


def from_reference(x):
    """A tpshift value (scenario, config, table, samples, ...) as this package's type."""
    import paper_2605_23945_b200 as pkg
    return _convert(x, pkg)


def to_reference(tpshift_module, x):
    """One of this package's decision-layer values as the reference's type."""
    return _convert(x, tpshift_module)
