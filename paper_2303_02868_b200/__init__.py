"""B200-native page-granular parameter/optimizer update (Angel-PTM,
arxiv 2303.02868) — a drop-in for the hot path of the reference ``hiermem``
package: page pools (hiermem/pagemem.py), the Adam/buffer update path
(hiermem/lockfree.py) and page sharding (hiermem/scheduler.py:59-76), with
the data plane in sm_100a CUDA (libhm_page.so).

The names re-exported here are the reference's (hiermem/__init__.py:8-74)
for that path; the update-path names load torch lazily on first use.
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

_LAZY = {
    "AdamHyper": "lockfree", "DelayModel": "lockfree", "GradMessage": "lockfree",
    "MasterState": "lockfree", "ParamBuffer": "lockfree", "ConservationLedger": "lockfree",
    "accumulate_gradient": "lockfree", "apply_update": "lockfree", "publish_params": "lockfree",
    "sweep": "lockfree", "ingest_sweep": "lockfree", "ingest": "lockfree",
    "ShardingModel": "sharding", "ShardedPageStep": "sharding",
    "FusedShardedPageStep": "sharding", "symmetric_alloc": "sharding",
    "HostMasterState": "swap", "swap_sweep": "swap", "SSDMasterState": "ssd", "ssd_sweep": "ssd",
    "DevicePageManager": "pages", "LockFreeRunner": "actors", "ScheduleExecutor": "executor",
    "PageLayout": "layout",
}

__version__ = "0.1.0"


def __getattr__(name):
    mod = _LAZY.get(name)
    if mod is None:
        raise AttributeError(f"module {__name__!r} has no attribute {name!r}")
    import importlib
    return getattr(importlib.import_module(f".{mod}", __name__), name)
