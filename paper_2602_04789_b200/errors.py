"""Exception types with the reference's names and ValueError base classes."""


class ZeroActiveRowError(ValueError):
    """A query-block row has no active key blocks (attention.py:99-100)."""


class EmptyActiveSetError(ValueError):
    """Softmax was asked to normalize over an empty active set (numerics.py:15-16)."""


class DegenerateScheduleError(ValueError):
    """The error-weight schedule cannot support a beta solve (planner.py:24-25)."""
