"""B200-native all-pairs engine (Rocket, arXiv:2009.04755) behind the reference's plugin API.

The hot path -- the pairwise compare over cached items -- runs as hand-written
sm_100a CUDA in ``librocket.so`` behind a C ABI (``include/rocket.h``); this
package is the Python host side that mirrors the reference's
``allpairs.apps.Application`` contract (/root/reference/pkg/src/allpairs/apps.py:74-125).
"""

from ._lib import lib  # noqa: F401  (fails loudly when librocket.so is missing)
from .errors import AppError, DeadlockError, MalformedInput, NoEvictableSlot, SlotOverflow  # noqa: F401

__all__ = ["AppError", "DeadlockError", "MalformedInput", "NoEvictableSlot", "SlotOverflow"]
