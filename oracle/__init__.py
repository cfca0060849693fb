"""CPU oracle (test infrastructure only -- see oracle/oracle.py header)."""
from .oracle import (appearances, vertex_terms, cost_terms, width_cost,  # noqa: F401
                     pairwise_contract, fix_index, contract_one, contract,
                     contract_sliced, brute_force, slice_digits)
