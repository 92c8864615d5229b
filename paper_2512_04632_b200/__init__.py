"""B200-native AOL-preconditioned Newton-Schulz ("Turbo-Muon", arxiv 2512.04632).

The compute path is libturbons.so (hand-written sm_100a CUDA: tcgen05/TMEM/TMA GEMM
engine with symmetric Gram/A^2 and fused AXPY epilogues, a fused AOL preconditioner, a
grouped launcher), reached through its C ABI (include/turbo_ns.h).  This package is the
thin Python binding plus the multi-GPU sharder.  Importing it loads the library and fails
loudly if it is missing: there is no CPU fallback.
"""
from ._lib import NSError, lib  # noqa: F401  (raises ImportError if libturbons.so is missing)
from .api import (default_coeffs, gram, launch_count, orthogonalize, orthogonalize_list,  # noqa: F401
                  muon_apply, poly, precondition, profile_enable, profile_read, read_flags, set_path, set_workspace,
                  shutdown, update,
                  workspace_size)
from .muon import DistributedTurboMuon, TurboMuon  # noqa: F401
from .parallel import (lpt_owners, make_plan, ns_flops, orthogonalize_host, orthogonalize_sharded,  # noqa: F401
                       reduce_scatter_owned)

__version__ = "0.1.0"
