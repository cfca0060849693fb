"""bench.py contract pieces that need no GPU: the reference arm's JSON line
(the driver runs `bench.py --impl reference`), the nonzero-slice list of the
headline workload, and the north-star fixtures' agreement with the slicer."""
import json
import os
import subprocess
import sys

import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_reference_arm_json_line():
    out = subprocess.run([sys.executable, os.path.join(REPO, "bench.py"), "--impl", "reference",
                          "--config", "cfg1_3reg50", "--steps", "2", "--warmup", "1"],
                         capture_output=True, text=True, timeout=600, cwd=REPO)
    assert out.returncode == 0, out.stderr[-2000:]
    line = json.loads([ln for ln in out.stdout.splitlines() if ln.startswith("{")][-1])
    assert line["impl"] == "reference"
    assert line["higher_is_better"] is True and line["unit"] == "TFLOP/s"
    for key in ("metric", "value", "n_gpus", "steps", "warmup", "ms_per_step", "config", "cpu_baseline", "e2e"):
        assert key in line, key
    assert line["cpu_baseline"]["kind"] == "port" and line["cpu_baseline"]["cores"] >= 1
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["e2e"]["value"] == line["value"]
    assert line["value"] > 0


def test_reference_arm_other_ranks_exit_quietly():
    env = dict(os.environ, RANK="1", WORLD_SIZE="2")
    out = subprocess.run([sys.executable, os.path.join(REPO, "bench.py"), "--impl", "reference",
                          "--config", "cfg1_3reg50"], capture_output=True, text=True, timeout=300,
                         cwd=REPO, env=env)
    assert out.returncode == 0
    assert not [ln for ln in out.stdout.splitlines() if ln.startswith("{")]


def test_nonzero_slice_list_matches_the_slice_set():
    from paper_2002_01935_b200.harness.workloads import load_workload
    with open(os.path.join(REPO, "benchdata", "cfg4_7x7_d40.slices.json")) as fh:
        rec = json.load(fh)
    tn, tree, ss, _ = load_workload(rec["workload"])
    assert float(rec["ws"]) == float(ss.Ws) and int(rec["d"]) == int(ss.d)
    ids = [int(x) for x in rec["ids"]]
    assert len(ids) >= 8 * 23 and len(set(ids)) == len(ids)  # 8 ranks x (3 warm-up + 20 timed)
    assert all(0 <= s < ss.d for s in ids)


@pytest.mark.parametrize("key", ["d24", "d40", "d40r", "d40g", "d40gr", "syc"])
def test_northstar_fixture_matches_the_slicer(key):
    from paper_2002_01935_b200.harness.workloads import load_workload
    from paper_2002_01935_b200.slicing import slice_assignment
    with open(os.path.join(REPO, "tests", "golden", "northstar_fixtures.json")) as fh:
        fx = json.load(fh)[key]
    tn, tree, ss, _ = load_workload(fx["workload"], ws=fx["ws"])
    assert list(ss.labels) == fx["sliced_labels"]
    assert int(ss.per_slice_cost) == fx["ops_per_slice"]
    for row in fx["slices"][:4]:
        asg = slice_assignment(tn, ss, row["slice"])
        assert [int(asg[lbl]) for lbl in ss.labels] == row["digits"]
