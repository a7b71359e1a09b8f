"""GPU harness CLI (paper_1907_02129_b200.cli): the reference's flag
surface and exit codes (cli.py:20-147) -- usage and suite errors exit 1
before any device work (CPU)."""

import json

import pytest

from paper_1907_02129_b200 import cli


@pytest.mark.parametrize("argv", [
    ["--suite", "resnet18", "--variants", "indirect,bogus"],
    ["--suite", "resnet18", "--variants", ","],
    ["--suite", "resnet18", "--reps", "0"],
    ["--suite", "resnet18", "--warmup", "-1"],
    ["--suite", "resnet18", "--batch", "0"],
    ["--suite", "resnet18", "--lambda", "fast"],
    ["--suite", "resnet18", "--no-such-flag"],
])
def test_usage_errors_exit_1(argv):
    with pytest.raises(SystemExit) as e:
        cli.main(argv)
    assert e.value.code == cli.EXIT_USAGE


def test_suite_errors_exit_1(tmp_path, capsys):
    assert cli.main(["--suite", str(tmp_path / "missing.json")]) == cli.EXIT_USAGE
    bad = tmp_path / "bad.json"
    bad.write_text(json.dumps({"version": 9, "shapes": []}))
    assert cli.main(["--suite", str(bad)]) == cli.EXIT_USAGE
    assert "unsupported suite schema version" in capsys.readouterr().err


def test_variant_spellings_match_reference():
    assert cli.VARIANT_FLAGS["indirect"] == "indirect"
    assert cli.VARIANT_FLAGS["gemm"] == "gemm_based"
    assert cli.VARIANT_FLAGS["gemm-only"] == "gemm_only"
