"""GPU parity: the B200 executor (through the C ABI) vs the CPU oracle and the
reference golden vectors.  Tolerance: complex64 execution vs complex128
reference, norm-wise relative error <= 1e-5 (north_star).  Random networks
(iid complex leaves) cancel heavily, so for them (check_close with the
network) the bound is 1e-5 * max(|ref|, 1e-2 * |.|-network value): an
absolute floor of 1e-7 times the value of the network with every entry
replaced by its modulus -- the scale of the forward error bound of a
complex64 sum-of-products (about 2u = 1.2e-7 of it per rounding).  Circuit
amplitudes use the plain relative error."""
import numpy as np
import pytest

import oracle
from conftest import arr_from_json, golden_cases
from _util import case_objects, rel_err
from paper_2002_01935_b200.executor import (SlicedPlan, contract, contract_sliced,
                                            AmplitudeEngine)
from paper_2002_01935_b200.refpkg import TensorNetwork, TensorNode
from paper_2002_01935_b200.harness import generators as gen
from paper_2002_01935_b200.harness.paths import best_greedy_tree, greedy_tree
from paper_2002_01935_b200.slicing import greedy_slice
from paper_2002_01935_b200.refpkg import metrics

pytestmark = pytest.mark.gpu
TOL = 1e-5


def abs_network(tn):
    return tn.replace(nodes=[TensorNode(nd.id, nd.indices, np.abs(nd.data)) for nd in tn.nodes])


def check_close(got, ref, tn=None, tree=None, S=()):
    got = np.asarray(got, dtype=np.complex128)
    ref = np.asarray(ref, dtype=np.complex128)
    err = np.linalg.norm((got - ref).ravel())
    scale = np.linalg.norm(ref.ravel())
    if tn is not None:
        absval, _, _ = oracle.contract_sliced(abs_network(tn), tree, S)
        scale = max(scale, 1e-2 * np.linalg.norm(np.asarray(absval).ravel()))
    assert err <= TOL * scale, (err, scale)


CASES = golden_cases()


@pytest.mark.parametrize("precision", ["fp32", "3xtf32", "tf32-bf16x"])
@pytest.mark.parametrize("case", CASES, ids=[c["name"] for c in CASES])
def test_golden_values(case, precision):
    tn, tree = case_objects(case)
    for ent in case["sliced"]:
        if "value" not in ent:
            continue
        S = tuple(ent["labels"])
        val, e10, ops = contract_sliced(tn, tree, S, precision=precision)
        assert ops == int(ent["Cs"])
        check_close(val, arr_from_json(ent["value"]), tn, tree, S)
        for sid, v in ent.get("per_slice", {}).items():
            got, _, _ = contract_sliced(tn, tree, S, slice_ids=range(int(sid), int(sid) + 1),
                                        precision=precision)
            check_close(got, arr_from_json(v), tn, tree, S)


@pytest.mark.parametrize("prec", [1, 2])
def test_gemm_kernel_vs_numpy(prec):
    import torch
    rng = np.random.default_rng(0)
    from paper_2002_01935_b200 import _native as nat
    lib = nat.load()
    for (b, m, n, k) in [(1, 128, 128, 16), (1, 256, 384, 64), (2, 200, 136, 40), (1, 1024, 512, 1000),
                         (3, 128, 256, 8), (1, 256, 128, 65536), (2, 130, 132, 20000)]:
        A = (rng.standard_normal((b, m, k)) + 1j * rng.standard_normal((b, m, k))).astype(np.complex64)
        B = (rng.standard_normal((b, n, k)) + 1j * rng.standard_normal((b, n, k))).astype(np.complex64)
        ta = torch.from_numpy(A).cuda()
        tb = torch.from_numpy(B).cuda()
        tc = torch.zeros((b, m, n), dtype=torch.complex64, device="cuda")
        nat.check(lib.tnx_gemm_c64(ta.data_ptr(), tb.data_ptr(), tc.data_ptr(), b, m, n, k, prec,
                                   torch.cuda.current_stream().cuda_stream))
        ref = np.einsum("bmk,bnk->bmn", A.astype(np.complex128), B.astype(np.complex128))
        got = tc.cpu().numpy()
        assert rel_err(got, ref) < (2e-6 if prec == 1 else 3e-6), (b, m, n, k, rel_err(got, ref))


@pytest.mark.parametrize("seed", range(12))
def test_random_hyper_networks(seed):
    tn = gen.random_hyper_network(8, 14, seed=100 + seed, max_rank=5)
    tree = greedy_tree(tn, seed=seed)
    ref, _, ops_ref = oracle.contract(tn, tree)
    val, _, ops = contract(tn, tree)
    assert ops == ops_ref
    check_close(val, ref, tn, tree)
    closed = [l for l in tn.index_table if l not in tn.output and tn.carriers(l)][:2]
    if closed:
        refs, _, _ = oracle.contract_sliced(tn, tree, closed)
        vs, _, _ = contract_sliced(tn, tree, closed)
        check_close(vs, refs, tn, tree, closed)
        vs2, _, _ = contract_sliced(tn, tree, closed, graph=False, hoist=False)
        check_close(vs2, refs, tn, tree, closed)


def test_circuit_amplitude_sliced_gemm_path():
    tn = gen.grid_circuit(5, 5, 20, seed=5)
    tree = best_greedy_tree(tn, trials=4)
    m = metrics(tree, tn)
    ss = greedy_slice(tree, tn, min(m.width, 22) - 2, restarts=2)
    ref, _, _ = oracle.contract_sliced(tn, tree, ss.labels, slice_ids=range(0, 4))
    plan = SlicedPlan(tn, tree, ss, gemm_min_macs=2 ** 16, direct_planes=False).bind()
    kinds = {v["kind"] for v in plan.vertex_info()}
    plan.run(0, 4)
    got = plan.result()
    assert rel_err(got, ref) <= TOL, rel_err(got, ref)
    # intermediate-level parity on slice 2 for every dependent vertex
    rec = {}
    from paper_2002_01935_b200.slicing import slice_assignment
    asg = slice_assignment(tn, ss, 2)
    oracle.contract_one(tn, tree, ss.labels, asg, record=rec)
    for v in [x["ssa"] for x in plan.vertex_info()][-40:]:
        labels, arr = plan.debug_vertex(2, v)
        ol, oarr = rec[v]
        oarr = np.transpose(oarr, [ol.index(l) for l in labels])
        assert rel_err(arr, oarr) <= TOL, (v, rel_err(arr, oarr))
    plan.close()
    print("kinds", kinds)


def test_full_amplitude_statevector_and_unitarity():
    for case in CASES:
        if "statevector_amplitude" not in case:
            continue
        tn, tree = case_objects(case)
        val, _, _ = contract(tn, tree)
        assert abs(val - complex(arr_from_json(case["statevector_amplitude"]))) <= TOL * abs(val)
    # open-leg circuit: sum_x |c_x|^2 = 1 with one plan reused across bitstrings
    tn = gen.grid_circuit(2, 3, 6, seed=2, simplify=False)
    # turn the closing projections into open legs
    nodes, out = [], []
    for nd in tn.nodes:
        if len(nd.indices) == 1 and nd.id >= len(tn.nodes) - 6:
            out.append(nd.indices[0])
            continue
        nodes.append(nd)
    open_tn = TensorNetwork([TensorNode(i, nd.indices, nd.data) for i, nd in enumerate(nodes)],
                            tn.index_table, tuple(out))
    from paper_2002_01935_b200.executor import _project
    tree = greedy_tree(_project(open_tn, "0" * 6))
    eng = AmplitudeEngine(open_tn, tree)
    total = 0.0
    for x in range(64):
        bits = format(x, "06b")
        total += abs(eng(bits)) ** 2
    eng.close()
    assert abs(total - 1.0) <= 1e-5


def test_multi_slice_ranges_and_accumulator():
    tn = gen.random_regular(30, 3, seed=3)
    tree = best_greedy_tree(tn, trials=2)
    labels = list(tn.index_table)[:4]
    plan = SlicedPlan(tn, tree, labels).bind()
    plan.run(0, 7)
    plan.run(7, 16)
    full = plan.result()
    ref, _, _ = oracle.contract_sliced(tn, tree, labels)
    assert rel_err(full, ref) <= TOL
    plan.reset()
    plan.run(3, 4)
    ref3, _, _ = oracle.contract_sliced(tn, tree, labels, slice_ids=[3])
    assert rel_err(plan.result(), ref3) <= TOL
    with pytest.raises(ValueError):
        plan.run(0, 17)
    plan.close()


def test_tiled_pack_matches_gather_pack():
    tn = gen.grid_circuit(5, 5, 24, seed=7)
    tree = best_greedy_tree(tn, trials=3)
    m = metrics(tree, tn)
    ss = greedy_slice(tree, tn, min(m.width, 23) - 1, restarts=1)
    vals = []
    for tiled in (True, False):
        plan = SlicedPlan(tn, tree, ss, gemm_min_macs=2 ** 14, tiled_pack=tiled).bind()
        assert plan.stats()["num_gemm"] > 0
        plan.run(0, min(plan.d, 4))
        vals.append(plan.result())
        plan.close()
    ref, _, _ = oracle.contract_sliced(tn, tree, ss.labels, slice_ids=range(0, min(ss.d, 4)))
    for v in vals:
        assert rel_err(v, ref) <= TOL


def test_direct_planes_fusion_matches_materialised():
    """GEMM->GEMM operand-plane fusion gives the same slice values as the
    fully materialised path (and dumps of fused vertices are refused)."""
    from paper_2002_01935_b200.harness.workloads import load_workload
    tn, tree, ss, _ = load_workload("cfg4p_7x7_d20", ws=21)
    vals = []
    for direct in (True, False):
        plan = SlicedPlan(tn, tree, ss, gemm_min_macs=2 ** 14, direct_planes=direct).bind()
        plan.run(0, 8)
        vals.append(plan.result())
        if direct:
            fused = [v["ssa"] for v in plan.vertex_info() if v["kind"] == "gemm_tc"]
            assert plan.stats()["num_gemm"] >= 2
        plan.close()
    assert rel_err(vals[0], vals[1]) <= 5e-6
    ref, _, _ = oracle.contract_sliced(tn, tree, ss.labels, slice_ids=range(0, 8))
    assert rel_err(vals[0], ref) <= TOL


def _two_tensor_net(xl, yl, out, seed=0):
    rng = np.random.default_rng(seed)
    labels = list(dict.fromkeys(list(xl) + list(yl)))
    tab = {l: 2 for l in labels}
    x = (rng.standard_normal((2,) * len(xl)) + 1j * rng.standard_normal((2,) * len(xl))) / 2 ** (len(xl) / 4)
    y = (rng.standard_normal((2,) * len(yl)) + 1j * rng.standard_normal((2,) * len(yl))) / 2 ** (len(yl) / 4)
    from paper_2002_01935_b200.refpkg import ContractionTree
    tn = TensorNetwork([TensorNode(0, xl, x), TensorNode(1, yl, y)], tab, tuple(out))
    return tn, ContractionTree((0, 1), [(0, 1)])


def test_dot_path_permuted_layouts():
    labels = [f"a{i}" for i in range(20)]
    rng = np.random.default_rng(1)
    yl = list(rng.permutation(labels))
    tn, tree = _two_tensor_net(labels, yl, ())
    plan = SlicedPlan(tn, tree, ()).bind()
    assert [v["kind"] for v in plan.vertex_info()] == ["dot"]
    plan.run()
    got = complex(plan.result())
    plan.close()
    ref, _, _ = oracle.contract(tn, tree)
    assert abs(got - ref) <= 1e-5 * max(abs(ref), 1e-3)


def test_small_k_contraction_on_tensor_cores():
    ml = [f"m{i}" for i in range(11)]
    nl = [f"n{i}" for i in range(10)]
    kl = ["k0", "k1"]
    tn, tree = _two_tensor_net(ml + kl, kl[::-1] + nl, ml + nl)
    plan = SlicedPlan(tn, tree, ()).bind()
    assert [v["kind"] for v in plan.vertex_info()] == ["gemm_tc"]
    plan.run()
    got = plan.result()
    plan.close()
    ref, _, _ = oracle.contract(tn, tree)
    assert rel_err(got, ref) <= 2e-6


def test_contract_cli_json(tmp_path):
    import json
    from paper_2002_01935_b200.refpkg import save_network
    from paper_2002_01935_b200.refpkg import tree_to_path_dict
    from paper_2002_01935_b200.contract_cli import main
    tn = gen.grid_circuit(4, 4, 10, seed=3)
    tree = best_greedy_tree(tn, trials=2)
    ss = greedy_slice(tree, tn, metrics(tree, tn).width - 2, restarts=1)
    save_network(tn, tmp_path / "n.json")
    (tmp_path / "p.json").write_text(json.dumps(tree_to_path_dict(tree, "ssa")))
    (tmp_path / "s.json").write_text(json.dumps(ss.to_dict()))
    import io, contextlib
    buf = io.StringIO()
    with contextlib.redirect_stdout(buf):
        rc = main([str(tmp_path / "n.json"), str(tmp_path / "p.json"), "--slices", str(tmp_path / "s.json")])
    assert rc == 0
    doc = json.loads(buf.getvalue())
    ref, _, ops = oracle.contract_sliced(tn, tree, ss.labels)
    got = complex(*doc["value"])
    assert abs(got - ref) <= 1e-5 * abs(ref)
    assert int(doc["op_count"]) == ops == ss.Cs


def test_batched_hyperedge_gemm():
    """Shared labels kept at the vertex (hyperedge / batch dims, dense.py:64-66)
    on the tensor-core path: z[b, m, n] = sum_k x[b, m, k] y[b, n, k]."""
    bl = ["b0", "b1"]
    ml = [f"m{i}" for i in range(8)]
    nl = [f"n{i}" for i in range(8)]
    kl = [f"k{i}" for i in range(6)]
    # batch labels also appear on a third (tiny) node so they are hyperedges kept at the pair
    rng = np.random.default_rng(5)
    xl, yl = bl + ml + kl, kl[::-1] + nl + bl[::-1]
    tab = {l: 2 for l in bl + ml + nl + kl}
    x = (rng.standard_normal((2,) * len(xl)) + 1j * rng.standard_normal((2,) * len(xl))) / 8
    y = (rng.standard_normal((2,) * len(yl)) + 1j * rng.standard_normal((2,) * len(yl))) / 8
    w = rng.standard_normal((2, 2)) + 0j
    from paper_2002_01935_b200.refpkg import ContractionTree
    tn = TensorNetwork([TensorNode(0, xl, x), TensorNode(1, yl, y), TensorNode(2, bl, w)], tab,
                       tuple(ml + nl))
    tree = ContractionTree((0, 1, 2), [(0, 1), (3, 2)])
    plan = SlicedPlan(tn, tree, ()).bind()
    info = plan.vertex_info()
    assert info[0]["kind"] == "gemm_tc" and info[0]["batch"] == 4
    plan.run()
    got = plan.result()
    plan.close()
    ref, _, _ = oracle.contract(tn, tree)
    assert rel_err(got, ref) <= 2e-6


def test_strip_exponent_beyond_fp32_range():
    """with strip_exponent every intermediate is renormalised
    on device, so a network whose value is far outside FP32 range contracts
    correctly; value * 10^exponent is invariant."""
    tn0 = gen.random_regular(40, 3, seed=9)
    # blow every leaf up by 1e6: value scales by 1e240 (beyond FP32 and FP64 range)
    tn = tn0.replace(nodes=[TensorNode(nd.id, nd.indices, nd.data * 1e6) for nd in tn0.nodes])
    tree = best_greedy_tree(tn0, trials=2)
    S = list(tn.index_table)[:3]
    ref0, _, _ = oracle.contract_sliced(tn0, tree, S)
    val, e10, _ = contract_sliced(tn, tree, S, {"strip_exponent": True})
    # compare log10 magnitudes and phases
    lg = np.log10(abs(val)) + e10
    lg_ref = np.log10(abs(ref0)) + 240
    assert abs(lg - lg_ref) < 1e-5
    assert abs(np.angle(val) - np.angle(ref0)) < 1e-4
    # plain mode overflows -> FloatingPointError, like the SPEC's non-finite check
    with pytest.raises(FloatingPointError):
        contract_sliced(tn, tree, S)
    # strip mode on an ordinary network agrees with plain mode
    v2, e2, _ = contract_sliced(tn0, tree, S, {"strip_exponent": True})
    assert abs(v2 * 10.0 ** e2 - ref0) <= 1e-5 * abs(ref0)


@pytest.mark.parametrize("dims", [(3, 5, 3), (3, 3, 5), (7, 3, 2)])
def test_gemm_path_odd_dims(dims):
    """Tensor-core path with non-power-of-two label dims: ragged M/N tiles,
    K padded to 16 (gather pack), division-based index maps, batch > 1."""
    dm, dn, dk = dims
    rng = np.random.default_rng(sum(dims))
    ml = ["m0", "m1", "m2", "m3", "m4"]
    nl = ["n0", "n1", "n2", "n3", "n4"]
    kl = ["k0", "k1", "k2"]
    tab = {**{l: dm for l in ml}, **{l: dn for l in nl}, **{l: dk for l in kl}, "b": 3}
    xl, yl = ml[:3] + kl + ["b"] + ml[3:], ["b"] + nl + kl[::-1]
    xs = tuple(tab[l] for l in xl)
    ys = tuple(tab[l] for l in yl)
    x = (rng.standard_normal(xs) + 1j * rng.standard_normal(xs)) / np.sqrt(np.prod(xs) ** 0.5)
    y = (rng.standard_normal(ys) + 1j * rng.standard_normal(ys)) / np.sqrt(np.prod(ys) ** 0.5)
    w = rng.standard_normal(3) + 0j
    from paper_2002_01935_b200.refpkg import ContractionTree
    tn = TensorNetwork([TensorNode(0, xl, x), TensorNode(1, yl, y), TensorNode(2, ["b"], w)], tab,
                       tuple(nl[:2] + ml + nl[2:]))
    tree = ContractionTree((0, 1, 2), [(0, 1), (3, 2)])
    plan = SlicedPlan(tn, tree, (), gemm_min_macs=1.0).bind()
    info = plan.vertex_info()
    assert info[0]["kind"] == "gemm_tc", info
    plan.run()
    got = plan.result()
    plan.close()
    ref, _, _ = oracle.contract(tn, tree)
    assert rel_err(got, ref) <= 2e-6, rel_err(got, ref)
    # sliced on a K label and a batch label
    val, _, _ = contract_sliced(tn, tree, ["k1", "b"])
    assert rel_err(val, ref) <= 2e-6


def test_edge_cases_single_leaf_hyperedge_dim1():
    from paper_2002_01935_b200.refpkg import from_arrays
    from paper_2002_01935_b200.refpkg import ContractionTree
    rng = np.random.default_rng(11)
    # single-node network, output subset, sliced dangling label
    a = rng.standard_normal((2, 3, 4)) + 1j * rng.standard_normal((2, 3, 4))
    tn = from_arrays("abc->ca", [a])
    tree = ContractionTree((0,), [])
    for S in ((), ("b",)):
        ref, _, _ = oracle.contract_sliced(tn, tree, S)
        got, _, ops = contract_sliced(tn, tree, S)
        assert rel_err(got, ref) <= 1e-6 and ops == 0
    # hyperedge label on three leaves, sliced; a dim-1 label; open output
    x = rng.standard_normal((2, 1, 3)) + 0j
    y = rng.standard_normal((2, 3, 2)) + 1j
    z = rng.standard_normal((2, 2)) - 1j
    tn = from_arrays("hqa,hab,hb->q", [x, y, z])
    tree = ContractionTree((0, 1, 2), [(0, 1), (3, 2)])
    for S in ((), ("h",), ("h", "a"), ("b",)):
        ref, _, _ = oracle.contract_sliced(tn, tree, S)
        got, _, _ = contract_sliced(tn, tree, S)
        assert rel_err(got, ref) <= 1e-6, S


def test_sliced_label_without_carrier_multiplies_by_dim():
    """A sliced index carried by no tensor contributes a factor d (every slice
    is identical) -- same as the oracle's slice loop."""
    from paper_2002_01935_b200.refpkg import TensorNetwork, TensorNode
    from paper_2002_01935_b200.refpkg import ContractionTree
    rng = np.random.default_rng(2)
    x = rng.standard_normal((2, 2)) + 0j
    y = rng.standard_normal((2, 2)) + 0j
    tn = TensorNetwork([TensorNode(0, "ab", x), TensorNode(1, "ba", y)], {"a": 2, "b": 2, "z": 3}, ())
    tree = ContractionTree((0, 1), [(0, 1)])
    ref, _, _ = oracle.contract_sliced(tn, tree, ["z"])
    got, _, _ = contract_sliced(tn, tree, ["z"])
    assert abs(got - ref) <= 1e-6 * abs(ref)
    assert abs(ref - 3 * np.trace(x @ y)) <= 1e-12 * abs(ref)


def test_large_sliced_leaves_gather():
    """Slice-dependent leaves of very different sizes in one gather launch
    (per-job block ranges), sliced labels between kept ones (no run merge
    across them) and mixed dims; every slice against the oracle."""
    from paper_2002_01935_b200.refpkg import ContractionTree
    rng = np.random.default_rng(5)
    tab = {"m0": 4, "s0": 2, "k0": 4, "m1": 4, "k1": 4, "m2": 512, "s1": 3, "n0": 8, "t": 2}
    shapes = {0: ["m0", "s0", "k0", "m1", "k1", "m2"], 1: ["k1", "s1", "k0", "n0"], 2: ["n0", "s1", "t"]}
    nodes = []
    for i, ls in shapes.items():
        shp = [tab[l] for l in ls]
        a = (rng.standard_normal(shp) + 1j * rng.standard_normal(shp)) / np.sqrt(np.prod(shp) ** 0.5)
        nodes.append(TensorNode(i, ls, a))
    tn = TensorNetwork(nodes, tab, ("m0", "m1", "m2", "t"))
    tree = ContractionTree((0, 1, 2), [(0, 1), (3, 2)])
    S = ("s0", "s1")
    plan = SlicedPlan(tn, tree, S).bind()
    assert plan.d == 6
    for s in range(6):
        plan.reset()
        plan.run(s, s + 1)
        ref, _, _ = oracle.contract_sliced(tn, tree, S, slice_ids=[s])
        assert rel_err(plan.result(), ref) <= TOL, s
    plan.reset()
    plan.run()
    ref, _, _ = oracle.contract_sliced(tn, tree, S)
    assert rel_err(plan.result(), ref) <= TOL
    plan.close()


def test_allreduce_plans_on_one_device():
    """tnx_allreduce over three plans (same GPU) holding disjoint slice blocks:
    every plan ends with the total, equal to the oracle's full sliced sum."""
    from paper_2002_01935_b200.executor import allreduce_plans
    tn = gen.grid_circuit(4, 4, 12, seed=3)
    tree = best_greedy_tree(tn, trials=2)
    ss = greedy_slice(tree, tn, metrics(tree, tn).width - 3, restarts=1)
    plans = [SlicedPlan(tn, tree, ss).bind() for _ in range(3)]
    try:
        d = plans[0].d
        assert d >= 3
        cuts = [0, d // 3, 2 * d // 3, d]
        for g, p in enumerate(plans):
            p.run(cuts[g], cuts[g + 1])
        allreduce_plans(plans)
        ref, _, _ = oracle.contract_sliced(tn, tree, ss.labels)
        vals = [p.result() for p in plans]
        for v in vals:
            assert rel_err(v, ref) <= TOL
        assert all(np.array_equal(vals[0], v) for v in vals[1:])
        # mismatched output size is refused
        tn2, tree2 = _two_tensor_net(["a", "b"], ["b", "c"], ["a", "c"])
        other = SlicedPlan(tn2, tree2, ()).bind()
        try:
            assert other.stats()["out_elements"] == 4 != plans[0].stats()["out_elements"]
            with pytest.raises(ValueError, match="output size"):
                allreduce_plans([plans[0], other])
        finally:
            other.close()
    finally:
        for p in plans:
            p.close()


@pytest.mark.parametrize("strip", [False, True])
def test_contract_sliced_device_list_sums_on_device(strip):
    """contract_sliced(devices=(0, 0)): two plans, one host thread each, the
    partials summed by tnx_allreduce (plain and strip_exponent modes)."""
    tn = gen.grid_circuit(4, 4, 12, seed=5)
    tree = best_greedy_tree(tn, trials=2)
    ss = greedy_slice(tree, tn, metrics(tree, tn).width - 2, restarts=1)
    opts = {"strip_exponent": strip}
    v2, e2, ops2 = contract_sliced(tn, tree, ss, opts, devices=(0, 0))
    v1, e1, ops1 = contract_sliced(tn, tree, ss, opts, devices=(0,))
    ref, _, _ = oracle.contract_sliced(tn, tree, ss.labels)
    assert ops1 == ops2 == ss.Cs
    got2 = np.asarray(v2) * 10.0 ** e2
    got1 = np.asarray(v1) * 10.0 ** e1
    assert rel_err(got2, ref) <= TOL and rel_err(got1, ref) <= TOL
    assert rel_err(got2, got1) <= 1e-12


def test_high_rank_sliced_leaf():
    """A rank-21 leaf carrying a sliced label (kept labels merge into two
    contiguous runs, so the gather's 16-run limit is not hit)."""
    from paper_2002_01935_b200.refpkg import ContractionTree
    rng = np.random.default_rng(11)
    al = [f"a{i}" for i in range(10)]
    bl = [f"b{i}" for i in range(10)]
    tab = {l: 2 for l in al + bl + ["s", "c"]}
    xl = al[:5] + ["s"] + al[5:] + bl          # rank 21, s in the middle
    yl = bl + ["s", "c"]
    x = ((rng.standard_normal((2,) * 21) + 1j * rng.standard_normal((2,) * 21)) / 32).astype(np.complex128)
    y = ((rng.standard_normal((2,) * 12) + 1j * rng.standard_normal((2,) * 12)) / 32).astype(np.complex128)
    tn = TensorNetwork([TensorNode(0, xl, x), TensorNode(1, yl, y)], tab, tuple(al + ["c"]))
    tree = ContractionTree((0, 1), [(0, 1)])
    got, _, _ = contract_sliced(tn, tree, ("s",))
    ref, _, _ = oracle.contract_sliced(tn, tree, ("s",))
    assert rel_err(got, ref) <= TOL


@pytest.mark.parametrize("dims", [dict(b=3, m=(4, 4, 4, 4, 4), n=(5, 5, 6), k=(3, 4, 2)),    # batched, N=150
                                  dict(b=1, m=(2,) * 11, n=(3, 3, 3, 3, 3), k=(2,) * 6)])  # N=243 (edge tile)
def test_stacked_b_gemm_shapes(dims):
    """The stacked-B 2-CTA GEMM (M >= 1024 rows of A): batched hyperedge
    labels, N not a multiple of the 128-column tile, K padded to 16."""
    from paper_2002_01935_b200.refpkg import ContractionTree
    rng = np.random.default_rng(21)
    bl = [f"h{i}" for i in range(1)] if dims["b"] > 1 else []
    ml = [f"m{i}" for i in range(len(dims["m"]))]
    nl = [f"n{i}" for i in range(len(dims["n"]))]
    kl = [f"k{i}" for i in range(len(dims["k"]))]
    tab = dict(zip(ml, dims["m"])) | dict(zip(nl, dims["n"])) | dict(zip(kl, dims["k"]))
    if bl:
        tab[bl[0]] = dims["b"]
    xl, yl = bl + ml + kl, kl[::-1] + nl + bl
    def rnd(ls):
        shp = [tab[l] for l in ls]
        return (rng.standard_normal(shp) + 1j * rng.standard_normal(shp)) / np.sqrt(np.prod([tab[l] for l in kl]))
    tn = TensorNetwork([TensorNode(0, xl, rnd(xl)), TensorNode(1, yl, rnd(yl))], tab, tuple(bl + ml + nl))
    tree = ContractionTree((0, 1), [(0, 1)])
    plan = SlicedPlan(tn, tree, ()).bind()
    assert [v["kind"] for v in plan.vertex_info()] == ["gemm_tc"]
    plan.run()
    got = plan.result()
    plan.close()
    ref, _, _ = oracle.contract(tn, tree)
    assert rel_err(got, ref) <= 2e-6


def test_stacked_parent_fed_by_direct_children():
    """A stacked-B parent GEMM whose B operand planes (incl. the negated
    imaginary planes) are written by a child GEMM's epilogue, vs the
    materialised path and the oracle."""
    from paper_2002_01935_b200.refpkg import ContractionTree
    rng = np.random.default_rng(8)
    al = [f"a{i}" for i in range(11)]
    kl = [f"k{i}" for i in range(7)]
    bl = [f"b{i}" for i in range(10)]
    jl = [f"j{i}" for i in range(5)]
    tab = {l: 2 for l in al + kl + bl + jl}
    def rnd(ls):
        shp = [2] * len(ls)
        return (rng.standard_normal(shp) + 1j * rng.standard_normal(shp)) / 2 ** (len(ls) / 4)
    # child = y[j, b] . z[j, k] -> [b, k];  parent = x[a, k] . child[b, k] -> [a, b]
    tn = TensorNetwork([TensorNode(0, al + kl, rnd(al + kl)), TensorNode(1, jl + bl, rnd(jl + bl)),
                        TensorNode(2, jl + kl, rnd(jl + kl))], tab, tuple(al + bl))
    tree = ContractionTree((0, 1, 2), [(1, 2), (0, 3)])
    vals = []
    for direct in (True, False):
        plan = SlicedPlan(tn, tree, (), gemm_min_macs=2 ** 10, direct_planes=direct).bind()
        plan.run()
        vals.append(plan.result())
        plan.close()
    ref, _, _ = oracle.contract(tn, tree)
    # two chained GEMMs; the parent's 8-k-block units run a 6-k-block first TMEM
    # round (TNX_GEMM_FIRST), so allow ~2e-6 per GEMM (north star: 1e-5)
    for v in vals:
        assert rel_err(v, ref) <= 5e-6


def test_amplitude_open_qubits_batch():
    """Bitstrings with open qubits ('x'): one contraction returns the
    amplitudes of all 2^N_f completions (PAPER.md N_f open qubits), equal to
    the individual full-bitstring amplitudes and the oracle."""
    from paper_2002_01935_b200.executor import _project, amplitude
    tn = gen.grid_circuit(2, 3, 6, seed=4, simplify=False)
    nodes, out = [], []
    for nd in tn.nodes:
        if len(nd.indices) == 1 and nd.id >= len(tn.nodes) - 6:
            out.append(nd.indices[0])
            continue
        nodes.append(nd)
    open_tn = TensorNetwork([TensorNode(i, nd.indices, nd.data) for i, nd in enumerate(nodes)],
                            tn.index_table, tuple(out))
    pattern = "0x1x00"
    ptn = _project(open_tn, pattern)
    tree = greedy_tree(ptn)
    eng = AmplitudeEngine(open_tn, tree, open_qubits=pattern)
    batch = np.asarray(eng(pattern))
    assert batch.shape == (2, 2)
    ref, _, _ = oracle.contract(ptn, tree)
    assert rel_err(batch, ref) <= TOL
    with pytest.raises(ValueError):
        eng("000000")
    eng.close()
    full_tree = greedy_tree(_project(open_tn, "0" * 6))
    full = AmplitudeEngine(open_tn, full_tree)
    for a in range(2):
        for b in range(2):
            c = full(f"0{a}1{b}00")
            assert abs(batch[a, b] - c) <= 1e-5 * max(abs(c), 1e-3)
    full.close()
    assert np.allclose(np.asarray(amplitude(open_tn, pattern, tree)), batch, atol=1e-7)


def test_amplitude_open_qubits_sliced():
    """Open qubits together with slicing: the (2, 2) amplitude tensor summed
    over slices (output permutation + tensor-valued accumulation) equals the
    unsliced oracle."""
    from paper_2002_01935_b200.executor import _project, amplitude
    tn = gen.grid_circuit(3, 4, 8, seed=6, simplify=False)
    nq = 12
    nodes, out = [], []
    for nd in tn.nodes:
        if len(nd.indices) == 1 and nd.id >= len(tn.nodes) - nq:
            out.append(nd.indices[0])
            continue
        nodes.append(nd)
    open_tn = TensorNetwork([TensorNode(i, nd.indices, nd.data) for i, nd in enumerate(nodes)],
                            tn.index_table, tuple(out))
    pattern = "x0110100101x"
    ptn = _project(open_tn, pattern)
    tree = best_greedy_tree(ptn, trials=2)
    ss = greedy_slice(tree, ptn, metrics(tree, ptn).width - 2, restarts=1)
    assert ss.d > 1
    got = np.asarray(amplitude(open_tn, pattern, tree, ss))
    ref, _, _ = oracle.contract(ptn, tree)
    assert got.shape == (2, 2)
    assert rel_err(got, ref) <= TOL
