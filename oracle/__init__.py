"""CPU oracle -- TEST INFRASTRUCTURE ONLY.

May be imported only by tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
--impl reference legs.  The product path (paper_2007_00202_b200) never imports it.
See oracle/dense.py for the definitions it implements and their PAPER.md citations.
"""
from .dense import (apply_op, bf_apply, bf_cols_apply_adj, bf_dense, bf_dense_tree, bf_extract,
                    bf_rows_apply, hodbf_apply, hodbf_dense, hodbf_dense_tree, hodbf_extract, hodbf_rows_apply,
                    rel_err, validate)

__all__ = ["apply_op", "bf_apply", "bf_cols_apply_adj", "bf_dense", "bf_dense_tree", "bf_extract",
           "bf_rows_apply", "hodbf_apply", "hodbf_dense", "hodbf_dense_tree", "hodbf_extract", "hodbf_rows_apply", "rel_err",
           "validate"]
