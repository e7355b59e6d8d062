"""Binding the reference package's hot path to this one.

`route_reference(kmf)` applies at run time what the two modules of
INTEGRATION.md (kmf/_b200.py for the solver, the build_stencils hook of
kmf/geometry.py) do when a `kmf` maintainer adds them: every name under
which the reference's modules reach the hot path -- `kmf.solve`,
`kmf.solver.solve`, `kmf.bench.solve`, `kmf.cli.solve` (validation.py goes
through `kmf.solver.solve`) -- runs this package's B200 `solve`, and
`build_stencils` the native bit-exact builder.

The reference's own harness (kmf.bench: BenchmarkReport, timed_run, sweep,
the JSON/CSV writers; bench.py:45-259) and CLI (kmf.cli generate / solve /
bench / validate / info; cli.py:112-292) then produce their own report
formats from B200 runs unchanged: this package does not restate them.
`solve` here accepts the reference's own SolverConfig, PointCloud,
Connectivity and Primitives (tests/test_dropin.py) and returns a
SolveResult with the reference's fields.

`unroute(kmf)` restores the reference's numpy path.
"""

from __future__ import annotations

import time

_SOLVE_HOLDERS = ("", "solver", "bench", "cli")        # modules that bound `solve` by name
_BUILD_HOLDERS = ("", "geometry", "bench", "cli")      # ... and `build_stencils`
_SAVED = "_b200_saved"


def _modules(kmf, names):
    for name in names:
        mod = kmf if not name else getattr(kmf, name, None)
        if mod is not None:
            yield mod


def route_reference(kmf, stencils: bool = True) -> None:
    """Route `kmf` (the imported reference package) to the B200 path."""
    import importlib

    for sub in ("solver", "geometry", "bench", "cli", "validation"):
        try:
            importlib.import_module(f"{kmf.__name__}.{sub}")
        except ImportError:
            pass
    from . import solver as _solver
    from .builder import build_stencils_native

    def solve(config, cloud, conn=None, initial_state=None, instrument=True, timing_skip=0,
              clock=time.perf_counter):
        """kmf.solver.solve (solver.py:477-573) on the B200."""
        return _solver.solve(config, cloud, conn, initial_state, instrument, timing_skip, clock)

    saved = getattr(kmf, _SAVED, None) or {}
    for mod in _modules(kmf, _SOLVE_HOLDERS):
        if hasattr(mod, "solve"):
            saved.setdefault((mod.__name__, "solve"), mod.solve)
            mod.solve = solve
    if stencils:
        for mod in _modules(kmf, _BUILD_HOLDERS):
            ref_build = getattr(mod, "build_stencils", None)
            if ref_build is None:
                continue
            saved.setdefault((mod.__name__, "build_stencils"), ref_build)

            def build_stencils(cloud, epsilon=None, k=None):
                """kmf.geometry.build_stencils (geometry.py:453-518) on the
                native bit-exact builder (k-nearest and radius modes)."""
                return build_stencils_native(cloud, k=k, epsilon=epsilon)

            mod.build_stencils = build_stencils
    setattr(kmf, _SAVED, saved)


def unroute(kmf) -> None:
    """Undo route_reference."""
    import sys

    saved = getattr(kmf, _SAVED, None) or {}
    for (modname, attr), fn in saved.items():
        mod = sys.modules.get(modname)
        if mod is not None:
            setattr(mod, attr, fn)
    if hasattr(kmf, _SAVED):
        delattr(kmf, _SAVED)


def main(argv=None) -> int:
    """`python -m paper_2108_07031_b200.integration <kmf CLI arguments>`: the
    reference's own CLI (kmf.cli.main, cli.py:275) on the B200 path; `kmf`
    must be importable (e.g. its install under baseline/_ref on PYTHONPATH)."""
    import importlib

    kmf = importlib.import_module("kmf")
    route_reference(kmf)
    return importlib.import_module("kmf.cli").main(argv)


if __name__ == "__main__":
    raise SystemExit(main())
