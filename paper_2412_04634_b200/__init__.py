"""B200-native (sm_100a) Neural Incident Radiance Cache hot path.

A drop-in for the NIRC path of the reference package ``nirclab``
(arXiv 2412.04634): same module names and signatures, with every hot
function executed by hand-written CUDA kernels behind the C ABI declared in
``include/nirc_b200.h`` (library ``libnirc_b200.so`` built in-tree).
"""

__version__ = "0.1.0"
