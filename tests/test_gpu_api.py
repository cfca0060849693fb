"""GPU tests of the public API contract: the reference's own objects in, SPEC
signatures, the data checks at the C-ABI boundary, cross-stream ordering,
slice-id lists, the CLI's strip_exponent and the norm_exponent factor."""
import json

import numpy as np
import pytest

import oracle
from _util import rel_err
from paper_2002_01935_b200 import refpkg
from paper_2002_01935_b200.executor import SlicedPlan, contract_sliced, amplitude, _project
from paper_2002_01935_b200.harness import generators as gen
from paper_2002_01935_b200.slicing import greedy_slice

pytestmark = pytest.mark.gpu
TOL = 1e-5


def _open_circuit(rows, cols, depth, seed):
    """Grid circuit whose final projections are removed: open legs = qubits."""
    tn = gen.grid_circuit(rows, cols, depth, seed=seed, simplify=False)
    nq = rows * cols
    nodes, out = [], []
    for nd in tn.nodes:
        if len(nd.indices) == 1 and nd.id >= len(tn.nodes) - nq:
            out.append(nd.indices[0])
            continue
        nodes.append(nd)
    return refpkg.TensorNetwork([refpkg.TensorNode(i, nd.indices, nd.data) for i, nd in enumerate(nodes)],
                                tn.index_table, tuple(out))


def test_reference_objects_end_to_end():
    """hypertn.TensorNetwork + a hypertn greedy_sample tree (drivers/greedy.py:144)
    straight into the executor, sliced, vs the oracle."""
    tn = gen.grid_circuit(5, 5, 16, seed=11)
    assert type(tn) is refpkg.network.TensorNetwork
    tree = refpkg.greedy_sample(tn, 1.0, 0.0, 0)
    assert type(tree) is refpkg.tree.ContractionTree
    m = refpkg.metrics(tree, tn)
    ss = greedy_slice(tree, tn, m.width - 3, restarts=1)
    val, e10, ops = contract_sliced(tn, tree, ss)
    ref, _, ops_ref = oracle.contract_sliced(tn, tree, ss.labels)
    assert ops == ops_ref == ss.Cs
    assert e10 == 0.0
    assert abs(val - ref) <= TOL * abs(ref), (val, ref)


def test_amplitude_spec_signature_without_tree():
    """SPEC.md:533 amplitude(circuit_tn, bitstring): the tree comes from the
    reference's greedy_sample, the slicing from the device memory."""
    open_tn = _open_circuit(3, 3, 8, seed=3)
    bits = "010011010"
    got = amplitude(open_tn, bits)
    ptn = _project(open_tn, bits)
    tree = refpkg.greedy_sample(ptn, 1.0, 0.0, 0)
    ref, _, _ = oracle.contract(ptn, tree)
    assert abs(got - ref) <= TOL * abs(ref)
    with pytest.raises(ValueError):
        amplitude(open_tn, "01")


def test_amplitude_applies_norm_exponent():
    """value = contraction * 10**norm_exponent (network.py:55-58)."""
    open_tn = _open_circuit(2, 3, 6, seed=4)
    bits = "010110"
    base = amplitude(open_tn, bits)
    scaled_tn = refpkg.TensorNetwork(open_tn.nodes, open_tn.index_table, open_tn.output, norm_exponent=3.0)
    scaled = amplitude(scaled_tn, bits)
    assert abs(scaled - 1e3 * base) <= 1e-6 * abs(1e3 * base)


def test_bind_rejects_wrong_sizes_and_dtypes():
    import torch
    tn = gen.random_regular(12, 3, seed=1)
    tree = refpkg.greedy_sample(tn, 1.0, 0.0, 0)
    plan = SlicedPlan(tn, tree, ())
    good = [np.ascontiguousarray(tn.node(n).data) for n in tree.leaves]
    bad = list(good)
    bad[3] = np.zeros(3, dtype=np.complex128)
    with pytest.raises(refpkg.DataError):
        plan.bind(leaf_arrays=bad)
    with pytest.raises(refpkg.DataError):
        plan.bind(leaf_arrays=good[:-1])
    dev = [torch.from_numpy(a.real.copy()).cuda() for a in good]          # float64: not complex
    with pytest.raises(refpkg.DataError):
        plan.bind(leaf_arrays=dev)
    dev = [torch.from_numpy(a).to(torch.complex64).cuda() for a in good]
    dev[0] = dev[0][..., :1]
    with pytest.raises(refpkg.DataError):
        plan.bind(leaf_arrays=dev)
    plan.close()


def test_noncontiguous_device_leaves_and_cross_stream_order():
    """Transposed (non-contiguous) CUDA leaves are copied and kept alive;
    bind on one stream and run/result on another order correctly."""
    import torch
    tn = gen.grid_circuit(4, 4, 12, seed=5)
    tree = refpkg.greedy_sample(tn, 1.0, 0.0, 0)
    S = greedy_slice(tree, tn, refpkg.metrics(tree, tn).width - 2, restarts=1).labels
    ref, _, _ = oracle.contract_sliced(tn, tree, S)
    leaves = []
    for nid in tree.leaves:
        a = torch.from_numpy(np.ascontiguousarray(tn.node(nid).data)).to(torch.complex64).cuda()
        big = torch.zeros(tuple(a.shape) + (2,), dtype=torch.complex64, device="cuda")
        big[..., 0] = a
        view = big[..., 0]                       # same values, stride 2: non-contiguous
        assert not view.is_contiguous()
        leaves.append(view)
    plan = SlicedPlan(tn, tree, S)
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    for _ in range(3):
        with torch.cuda.stream(s1):
            plan.bind(leaf_arrays=leaves, stream=s1)
        plan.run(stream=s2)
        got = complex(plan.result(stream=torch.cuda.Stream()))
        assert abs(got - ref) <= TOL * abs(ref)
    plan.close()


def test_slice_id_list_semantics():
    """slice_ids is a list of ids, as in the oracle: [0, 7] is {0, 7}."""
    tn = gen.grid_circuit(4, 4, 10, seed=2)
    tree = refpkg.greedy_sample(tn, 1.0, 0.0, 0)
    ss = greedy_slice(tree, tn, refpkg.metrics(tree, tn).width - 3, restarts=1)
    assert ss.d >= 8
    ids = [0, 7, 3, 4, 5]
    got, _, ops = contract_sliced(tn, tree, ss, slice_ids=ids)
    ref, _, ops_ref = oracle.contract_sliced(tn, tree, ss.labels, slice_ids=ids)
    assert ops == ops_ref
    scale = sum(abs(oracle.contract_sliced(tn, tree, ss.labels, slice_ids=[i])[0]) for i in ids)
    assert abs(got - ref) <= TOL * scale
    with pytest.raises(ValueError):
        contract_sliced(tn, tree, ss, slice_ids=[ss.d])
    with pytest.raises(ValueError):
        contract_sliced(tn, tree, ss, slice_ids=range(0, 4, 2))


def test_cli_strip_exponent(tmp_path, capsys):
    """--strip-exponent renormalises every intermediate: a
    network whose value is ~1e240 contracts through the CLI."""
    from paper_2002_01935_b200.contract_cli import main
    tn0 = gen.random_regular(40, 3, seed=9)
    tn = tn0.replace(nodes=[refpkg.TensorNode(nd.id, nd.indices, nd.data * 1e6) for nd in tn0.nodes])
    tree = refpkg.greedy_sample(tn0, 1.0, 0.0, 0)
    refpkg.save_network(tn, str(tmp_path / "n.json"))
    (tmp_path / "p.json").write_text(json.dumps(refpkg.tree_to_path_dict(tree, "ssa")))
    rc = main([str(tmp_path / "n.json"), str(tmp_path / "p.json"), "--strip-exponent"])
    assert rc == 0
    doc = json.loads(capsys.readouterr().out)
    val = complex(*doc["value"])
    ref0, _, _ = oracle.contract(tn0, tree)
    assert abs(np.log10(abs(val)) + doc["exponent10"] - (np.log10(abs(ref0)) + 240)) < 1e-5
    # without the flag the value overflows: exit code 5 (numeric)
    assert main([str(tmp_path / "n.json"), str(tmp_path / "p.json")]) == 5


def test_measurement_diagnostics():
    """tnx_mma_peak (the roofline denominator) and tnx_clock_stamp (the clock
    the roofline is priced at) return physically plausible numbers."""
    import torch
    from paper_2002_01935_b200 import _native as nat
    sms = torch.cuda.get_device_properties(0).multi_processor_count
    for kind, cg, per_clk in (("tf32", 2, 4096), ("tf32", 1, 4096), ("bf16", 2, 8192), ("ffma", 1, 256)):
        t, mhz, ms = nat.mma_peak(kind, cg, 20000)
        assert 300 <= mhz <= 2500, (kind, mhz)
        rate = t * 1e12 / (mhz * 1e6) / sms  # flop per clock per SM
        assert 0.85 * per_clk <= rate <= 1.02 * per_clk, (kind, cg, rate)
        assert ms > 0
    with pytest.raises(ValueError):
        nat.mma_peak("tf32", 3, 20000)
    st = torch.cuda.Stream()
    stamps = nat.ClockStamps()
    stamps.start(st.cuda_stream)
    with torch.cuda.stream(st):
        a = torch.randn(4096, 4096, device="cuda")
        for _ in range(20):
            a = a @ a * 1e-2
    stamps.stop(st.cuda_stream)
    torch.cuda.synchronize()
    mhz, n = stamps.mhz()
    assert n >= sms // 2 and 300 <= mhz <= 2500, (mhz, n)


def test_run_slice_ids_matches_ranges():
    """tnx_run_slice_ids (any order, repeats, consecutive runs) sums exactly
    what the equivalent ranges do; out-of-range ids raise ValueError."""
    tn = gen.grid_circuit(4, 5, 12, seed=11)
    tree = refpkg.greedy_sample(tn, 1.0, 0.0, 0)
    ss = greedy_slice(tree, tn, refpkg.metrics(tree, tn).width - 4, restarts=1)
    plan = SlicedPlan(tn, tree, ss).bind()
    try:
        d = plan.d
        ids = [3, 4, 5, 0, 9 % d, 3]
        plan.reset()
        plan.run_ids(ids)
        got = complex(plan.result())
        plan.reset()
        for s in ids:
            plan.run(s, s + 1)
        ref = complex(plan.result())
        assert got == ref, (got, ref)
        with pytest.raises(ValueError):
            plan.run_ids([0, d])
        plan.reset()
        plan.run_ids([])
        assert complex(plan.result()) == 0
    finally:
        plan.close()


def test_result_async_matches_result():
    """tnx_partial_result_async enqueues the read; after a stream sync the
    buffer equals tnx_partial_result's value."""
    import torch
    tn = gen.grid_circuit(4, 4, 10, seed=5)
    tree = refpkg.greedy_sample(tn, 1.0, 0.0, 0)
    ss = greedy_slice(tree, tn, refpkg.metrics(tree, tn).width - 2, restarts=1)
    plan = SlicedPlan(tn, tree, ss).bind()
    try:
        st = torch.cuda.Stream()
        buf = torch.zeros(2, dtype=torch.float64).pin_memory()
        plan.run(0, plan.d, st)
        plan.result_async(buf, st)
        st.synchronize()
        ref = complex(plan.result(st))
        assert complex(buf[0].item(), buf[1].item()) == ref
        with pytest.raises(ValueError):
            plan.result_async(torch.zeros(1, dtype=torch.float64).pin_memory(), st)
    finally:
        plan.close()
