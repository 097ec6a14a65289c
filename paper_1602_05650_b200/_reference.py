"""The reference package (`slenderflow`) as a dependency of this one.

The north_star keeps the host-side logic in the reference's own Python
package; this package replaces its hot path (the HI operator, the block
rows, the preconditioner, GMRES and the state update) and calls back into
the reference for the scalar host logic it does not restate:

* dynamic-instability kinetics and the cortical contact models after a
  step (slenderflow.fiber.growth_rate / polymerization_step,
  slenderflow.system.cortical_push_update / cortical_pull_catastrophe;
  solver.py:574-588 of the reference), which none of the BASELINE configs
  enables;
* the nearest-point search on a surface profile R(theta)
  (slenderflow.body.nearest_surface_point, body.py:371-423) for targets in a
  surface's near shell, whose O(N_fine) map sums then run on the device.

Resolution order: an importable `slenderflow` (the reference installed as a
package), then this repository's staged copy in baseline/_ref (installed
unmodified by __graft_entry__.build(), which travels with the repository
snapshot).  Nothing on the all-pairs / matvec / GMRES path imports it.
"""

import importlib
import os
import sys

_STAGED = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                       "baseline", "_ref")


class ReferenceUnavailable(ImportError):
    pass


def module(name):
    """slenderflow.<name> (fiber, body, system, ...)."""
    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache_slenderflow")
    try:
        return importlib.import_module(f"slenderflow.{name}")
    except ImportError:
        pass
    if os.path.isdir(os.path.join(_STAGED, "slenderflow")):
        if _STAGED not in sys.path:
            sys.path.append(_STAGED)
        return importlib.import_module(f"slenderflow.{name}")
    raise ReferenceUnavailable(
        "this operation runs the reference's own host code (slenderflow): install it, or run "
        "__graft_entry__.build() to stage it in baseline/_ref")
