"""Shared helpers for tests (fixture decoding)."""
from paper_2002_01935_b200.refpkg import network_from_dict
from paper_2002_01935_b200.refpkg import ContractionTree


def case_objects(case):
    tn = network_from_dict(case["network"]) if "network" in case else None
    tree = ContractionTree(case["tree"]["leaves"], [tuple(p) for p in case["tree"]["pairs"]])
    return tn, tree


def rel_err(a, b):
    import numpy as np
    a = np.asarray(a, dtype=np.complex128)
    b = np.asarray(b, dtype=np.complex128)
    nb = np.linalg.norm(b.ravel())
    if nb == 0:
        return float(np.linalg.norm(a.ravel()))
    return float(np.linalg.norm((a - b).ravel()) / nb)
