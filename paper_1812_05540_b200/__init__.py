"""B200-native two-stage (fixed-stress + CPR) preconditioner inside FGMRES for
the coupled multiphase poromechanics Jacobian (arXiv 1812.05540).

The product is libtsp.so (CUDA sm_100a kernels + C-ABI, include/tsp.h); this
package only holds it and a ctypes binding (tsp.py)."""
from .tsp import (TSP_SETUP_FLOW, TSP_SETUP_MECH, Tsp, TspError, default_options,  # noqa: F401
                  lib, LIB_PATH, EXPORTED)
