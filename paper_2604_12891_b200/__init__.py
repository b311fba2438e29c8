"""paper_2604_12891_b200 -- B200-native (sm_100a) batched scorer of TCL's Mamba cost model.

Hot path: libtcl.so (csrc/, C ABI in include/tcl.h); Python binding: tcl.py.
"""
from .tcl import (Model, TclError, load, tcl_comm_unique_id, tcl_dims, tcl_weights_count,  # noqa: F401
                  TCL_PREC_FP32, TCL_PREC_BF16_PROJ, TCL_DISC_ZOH, TCL_DISC_EULER_B)
