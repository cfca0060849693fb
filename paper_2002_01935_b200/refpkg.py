"""The reference package ``hypertn`` -- the layer this executor plugs under.

north_star keeps the reference's data model, tree layer and path finding as
they are ("the reference's contraction-tree / per-slice contract entry points
are kept so the GPU executor is a drop-in"), so this package does not carry
its own copy of them: ``TensorNetwork`` / ``TensorNode`` / ``DataError``
(`/root/reference/pkg/src/hypertn/network.py:18-136`), ``ContractionTree`` /
``annotate_incidence`` / ``metrics`` / path documents (`tree.py:32-223`),
``HyperView`` (`hypergraph.py:12-131`) and the drivers are imported from the
installed reference.

Where it comes from, first hit wins:

1. an already importable ``hypertn``;
2. ``<repo>/baseline/_ref`` -- the unmodified reference installed with
   ``pip install --no-index --target baseline/_ref`` (``build()`` does this in
   the build container; the directory travels to the GPU box with the repo);
3. ``/root/reference/pkg/src`` (build container only).

If none exists the import fails loudly -- there is no fallback copy.
"""

from __future__ import annotations

import importlib
import os
import sys

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF_INSTALL = os.path.join(REPO, "baseline", "_ref")
REF_SOURCE = "/root/reference/pkg/src"


def _locate():
    try:
        return importlib.import_module("hypertn.network")
    except ImportError:
        pass
    for path in (REF_INSTALL, REF_SOURCE):
        if os.path.isdir(os.path.join(path, "hypertn")):
            if path not in sys.path:
                sys.path.append(path)
            importlib.invalidate_caches()
            return importlib.import_module("hypertn.network")
    raise ImportError(
        "the reference package 'hypertn' is not importable: install it with "
        "`python -m pip install --no-index --no-build-isolation --no-deps "
        f"--target {REF_INSTALL} <copy of /root/reference/pkg>` (build() does this)")


network = _locate()
tree = importlib.import_module("hypertn.tree")
dense = importlib.import_module("hypertn.dense")
hypergraph = importlib.import_module("hypertn.hypergraph")
greedy = importlib.import_module("hypertn.drivers.greedy")
optimal = importlib.import_module("hypertn.drivers.optimal")

TensorNetwork = network.TensorNetwork
TensorNode = network.TensorNode
DataError = network.DataError
ContractionTree = tree.ContractionTree
annotate_incidence = tree.annotate_incidence
metrics = tree.metrics
HyperView = hypergraph.HyperView


def ordered_labels(tr, tn, v):
    """Labels of SSA vertex ``v`` in the reference's natural order: the key
    order of ``annotate_incidence``'s count dict (`tree.py:155-166`,
    `hypergraph.py:106-119`), which is also ``pairwise_contract``'s output
    order (`dense.py:74-75`)."""
    annotate_incidence(tr, tn)
    names = tr._ann.view.labels
    return tuple(names[li] for li in tr._ann.counts[v])


def install(dest=REF_INSTALL, source=os.path.dirname(REF_SOURCE), quiet=True):
    """Install the unmodified reference into ``dest`` (offline; the source is
    copied to /tmp first because /root/reference is read-only)."""
    import shutil
    import subprocess
    import tempfile
    if os.path.isdir(os.path.join(dest, "hypertn")):
        return dest
    if not os.path.isdir(source):
        raise FileNotFoundError(f"reference source {source} not found")
    tmp = tempfile.mkdtemp(prefix="hypertn_src_")
    src = os.path.join(tmp, "pkg")
    shutil.copytree(source, src)
    for root, dirs, files in os.walk(src):
        for f in dirs + files:
            os.chmod(os.path.join(root, f), 0o755)
    cmd = [sys.executable, "-m", "pip", "install", "--no-index", "--no-build-isolation", "--no-deps",
           "--find-links", "/opt/wheelhouse", "--target", dest, src]
    res = subprocess.run(cmd, capture_output=True, text=True)
    shutil.rmtree(tmp, ignore_errors=True)
    if res.returncode != 0:
        raise RuntimeError("installing the reference failed:\n" + res.stdout[-2000:] + res.stderr[-2000:])
    return dest


# names the harness, CLI and tests use, re-exported from the reference modules
network_from_dict = network.network_from_dict
network_to_dict = network.network_to_dict
from_arrays = network.from_arrays
parse_einsum_spec = network.parse_einsum_spec
save_network = network.save_network
load_network = network.load_network
validate = network.validate
tree_to_path_dict = tree.tree_to_path_dict
tree_from_path_dict = tree.tree_from_path_dict
minfill_order = tree.minfill_order
tree_from_edge_order = tree.tree_from_edge_order
greedy_sample = greedy.greedy_sample
