"""B200-native hot path of ARRABIT-MPM (Wen & Zhang, arXiv 1507.06078).

The product is ``libarrabit.so`` (C-ABI in ``include/arrabit.h``; CUDA for
sm_100a in ``csrc/``).  This package is its thin Python binding: it loads the
library on import and fails loudly if it is missing — there is no CPU path.
"""
from . import _lib
from .api import (  # noqa: F401
    ArrError,
    Comm,
    DeviceCSR,
    ColSplitContext,
    EigContext,
    eig_init,
    eig_init_colsplit,
    eig_solve_host,
    to_device_csr,
)

from . import partition  # noqa: F401,E402

LIB = _lib.load()
