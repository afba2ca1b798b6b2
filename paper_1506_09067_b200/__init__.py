"""B200-native (sm_100a) CHAOS hot path: controlled-hogwild CNN training behind a C ABI.

The product is ``libchaos.so`` (``csrc/``, ABI in ``include/chaos.h``); ``chaos`` is its
thin ctypes binding and ``dist`` the torch.distributed plumbing for multi-GPU weight
averaging.  Importing this package never touches ``oracle/``.
"""
from .chaos import (CHAOS_CONV, CHAOS_FULL, CHAOS_IDENTITY, CHAOS_MAXPOOL, CHAOS_TANH, HOGWILD, SYNC,  # noqa: F401
                    OPT_DEBUG_CLAIMS, OPT_DEBUG_STAGGER, OPT_DEBUG_TRACE, OPT_GROUP, OPT_MAX_CTAS, OPT_PAVG_COMM_CTAS,
                    OPT_RESERVE_SMS, OPT_STREAM, OPT_SYNC_BATCH,
                    ChaosError, Net, lib)
