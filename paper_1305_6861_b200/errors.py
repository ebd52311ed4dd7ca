"""Exception types of the host layer — same names and roles as the reference's
``mrsim.errors`` (errors.py:1-62), plus :class:`DeviceError` for CUDA failures.

C-ABI status codes map as follows (include/bloch_b200.h):

* ``BLOCH_E_INVALID`` -> :class:`InvalidParameter`  (engine.py:467-473)
* ``BLOCH_E_CUDA``    -> :class:`WorkerPanic`       (engine.py:575-577; errors.py:57-62)
* ``BLOCH_E_STATE`` / ``BLOCH_E_NOMEM`` -> :class:`DeviceError`
"""


class MrSimError(Exception):
    """Base class for all simulator errors (errors.py:4-5)."""


class InvalidParameter(MrSimError):
    """A numeric argument is outside its admissible range (errors.py:8-9)."""


class TimingInfeasible(MrSimError):
    """A sequence builder was asked for intervals that come out negative."""


class ParseError(MrSimError):
    """A file or description violates its format (errors.py:16-27)."""


class TrajectoryMismatch(MrSimError):
    """Echo records and trajectory metadata disagree in shape (errors.py:49-50)."""


class FitDiverged(MrSimError):
    """A relaxometry fit failed to converge (errors.py:53-54)."""


class SpinBudgetExceeded(MrSimError):
    """Rasterization would produce more spins than the configured cap."""


class WorkerPanic(MrSimError):
    """The device failed while processing a spin block (errors.py:57-62).

    ``block_index`` is the block (or, for the multi-GPU path, the rank) that
    failed; the message carries the library's error text.
    """

    def __init__(self, block_index, cause):
        self.block_index = block_index
        super().__init__(f"worker failed on block {block_index}: {cause}")


class DeviceError(MrSimError):
    """The CUDA engine is unavailable or was called out of order."""
