"""contract CLI error paths (SPEC.md:664 exit codes) -- no GPU needed."""
import json

from paper_2002_01935_b200.contract_cli import main


def test_usage_error_exit_2():
    assert main([]) == 2


def test_data_error_exit_4(tmp_path):
    (tmp_path / "bad.json").write_text(json.dumps({"indices": {"a": 2}, "output": ["zz"], "tensors": []}))
    (tmp_path / "p.json").write_text(json.dumps({"format": "ssa", "path": []}))
    assert main([str(tmp_path / "bad.json"), str(tmp_path / "p.json")]) == 4


def test_bad_path_exit_2(tmp_path):
    (tmp_path / "n.json").write_text(json.dumps({"indices": {"a": 2}, "output": [],
                                                  "tensors": [{"id": 0, "indices": ["a"], "data": None},
                                                              {"id": 1, "indices": ["a"], "data": None}]}))
    (tmp_path / "p.json").write_text(json.dumps({"format": "linear", "path": [[0, 5]]}))
    assert main([str(tmp_path / "n.json"), str(tmp_path / "p.json")]) == 2
