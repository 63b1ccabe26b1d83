"""B200-native FETI dual-operator engine (arxiv 2111.11728 hot path).

The product is ``lib/libfetigpu.so`` (CUDA C++ for sm_100a behind the C-ABI
in ``include/fetigpu.h``); :mod:`.engine` is its Python mirror of the
reference's solver entry points and :mod:`.problems` the seeded generators of
BASELINE.json's configs.
"""
from . import problems  # noqa: F401
from .problems import Problem, CONFIGS  # noqa: F401
