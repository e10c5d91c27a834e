"""Exception types of the reference API, re-declared for the B200 engine.

Names and meaning follow the reference package so callers' ``except``
clauses keep working:

* ``CapacityError``        -- gpu/layout.py:99-100 (buffers exceed the device)
* ``CollisionBudgetError`` -- collision.py:43-44 (pairs per frame over budget)
* ``AdapterUnavailable``   -- gpu/device.py:40-41 (no usable compute adapter)
* ``DivergenceError``      -- solver.py:44-45 (state stopped being finite)
"""


class CapacityError(RuntimeError):
    """The buffer layout does not fit the device."""


class CollisionBudgetError(RuntimeError):
    """Raised when a frame would exceed the configured pair-test budget."""


class AdapterUnavailable(RuntimeError):
    """No usable compute adapter for the requested backend."""


class DivergenceError(RuntimeError):
    """Raised when a node's state stops being finite."""
