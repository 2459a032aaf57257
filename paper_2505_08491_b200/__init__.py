"""B200-native (sm_100a) hot path of the neural-preconditioned FGMRES solve
for coupled 3D-1D systems (arXiv 2505.08491), a drop-in for the reference
``mdprec`` package's solve path: problem build, preconditioner objects and
the FGMRES solve call keep their names, arguments and error behaviour;
the arithmetic runs in hand-written CUDA kernels behind a C ABI
(include/mdp_b200.h, lib/libmdp_b200.so).
"""

__version__ = "0.1.0"
