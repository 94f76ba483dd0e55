"""B200-native swap hot path of Chameleon (arxiv 2509.11076): policy execution (batched
swap-out/in between HBM and mapped pinned host memory) and policy evaluation (candidate swap-set
replay), behind the C ABI in include/chm.h.  `chm` is the thin ctypes binding."""
from . import chm  # noqa: F401
from .chm import Context, Trace, ChmError, best_reduce, record_iteration, load  # noqa: F401
