"""B200-native two-stage (fixed-stress + CPR) preconditioner inside FGMRES for
the coupled multiphase poromechanics Jacobian (arXiv 1812.05540).

The product is libtsp.so (CUDA sm_100a kernels + C-ABI, include/tsp.h); this
package only holds it and a ctypes binding (tsp.py)."""
from .tsp import (TSP_COMM_LOCAL, TSP_COMM_NCCL, TSP_COMM_NONE, TSP_SETUP_FLOW, TSP_SETUP_MECH, TSP_SETUP_REFRESH,  # noqa: F401
                  AssembledProblem, EXPORTED, LIB_PATH, LocalWorld, Tsp, TspError, assemble, default_options, lib, masses, residual,
                  nccl_unique_id, partition)
