"""paper_2305_16432_b200 -- B200-native NeuralPCG solve path.

Drop-in for the reference package ``pcgkit``'s solve path
(``gnn.build_learned`` + ``pcg.pcg_solve``): the same module / class /
function names, argument meaning and exceptions, running on hand-written
sm_100a kernels in ``libnpcg.so`` (C ABI: include/npcg.h).
"""
__version__ = "0.1.0"

from . import errors  # noqa: F401
