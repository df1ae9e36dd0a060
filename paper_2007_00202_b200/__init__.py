"""B200-native multi-RHS butterfly / HOD-BF apply (arxiv 2007.00202 hot path).

The compute lives in libbfapply.so (include/bfapply.h, csrc/*.cu, sm_100a); this
package is the thin binding.  See DESIGN.md.
"""
from .bfapply import (BFError, BFHandle, HODBFHandle, bf_apply, bf_apply_adj, bf_apply_op, bf_create,
                      hodbf_apply, hodbf_create, lib, version)

__all__ = ["BFError", "BFHandle", "HODBFHandle", "bf_apply", "bf_apply_adj", "bf_apply_op", "bf_create",
           "hodbf_apply", "hodbf_create", "lib", "version"]
