"""Implicit coupled stepping on the device (solver.py of the reference)."""

import numpy as np


def host_elastic_force_density(fib, Xcand, Tcand):
    """f = -E Ds^4 X + Ds (T X_s) with frozen geometry (fiber.py:237-241).

    Host helper for API defaults (complementary_velocities with no explicit
    forces); the solver evaluates it on the device.
    """
    Ds, Ds2, _ = fib.ds_powers()
    Ds4 = Ds2 @ Ds2
    Xcand = np.asarray(Xcand, dtype=float)
    Tcand = np.asarray(Tcand, dtype=float)
    return -fib.E * (Ds4 @ Xcand) + Ds @ (Tcand[:, None] * fib.tangents)
