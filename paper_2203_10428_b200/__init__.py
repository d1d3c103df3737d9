"""B200-native PipeGCN training step (arXiv 2203.10428).

The hot path lives in libpgcn.so (csrc/, sm_100a kernels behind the C ABI of include/pgcn.h);
`pgcn` is the thin ctypes binding.  Build with `python -m paper_2203_10428_b200.build`.
"""
from . import pgcn  # noqa: F401
from .pgcn import Context, Partitioning, flatten_params, make_config, param_count, partition, unflatten_params  # noqa: F401
