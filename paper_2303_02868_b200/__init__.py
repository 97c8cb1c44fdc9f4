"""B200-native page-granular parameter/optimizer update (Angel-PTM,
arxiv 2303.02868) — a drop-in for the hot path of the reference ``hiermem``
package: page pools (hiermem/pagemem.py) and the Adam/buffer update path
(hiermem/lockfree.py), with the data plane in sm_100a CUDA (libhm_page.so).
"""
from .errors import AllocationError, ConfigError, MoveError, NativeError, ProtocolError
from .pagemem import (
    MIN_PAGE_BYTES,
    NOT_READY,
    PAGE_BYTES_DEFAULT,
    ManagedTensor,
    Occupant,
    Page,
    PageManager,
    PoolStats,
    Tier,
    TierPool,
    TransferDescriptor,
    fragmentation,
    pool_init,
    tensor_allocate,
    tensor_release,
)
from .workloads import TensorSpec

__version__ = "0.1.0"
