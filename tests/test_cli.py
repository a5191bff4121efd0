"""CLI front end (paper_2108_10470_b200/cli.py) -- the reference's
tests/test_cli.py contract: config validation exits 2, bench CSV columns and
constant-experience arithmetic.  The commands themselves need a GPU
(tests/test_gpu_ppo.py)."""

import pytest

from paper_2108_10470_b200 import cli


def test_unknown_config_section_and_key_exit_2(tmp_path, capsys):
    bad = tmp_path / "c.yaml"
    bad.write_text("trainer: {}\n")
    assert cli.main(["bench", "--env", "quadruped", "--config", str(bad)]) == 2
    bad.write_text("env:\n  num_env: 3\n")
    assert cli.main(["bench", "--env", "quadruped", "--config", str(bad)]) == 2
    bad.write_text("ppo:\n  lrr: 3\n")
    assert cli.main(["train", "--env", "quadruped", "--config", str(bad)]) == 2
    bad.write_text(": : :\n")
    assert cli.main(["train", "--env", "quadruped", "--config", str(bad)]) == 2
    assert cli.main(["train", "--env", "quadruped", "--config", str(tmp_path / "missing.yaml")]) == 2
    assert "config error" in capsys.readouterr().err


def test_env_counts_parsing():
    assert cli._parse_env_counts("64, 256,1024") == [64, 256, 1024]
    for bad in ("", "a,b", "0,4", "-1"):
        with pytest.raises(cli.ConfigError):
            cli._parse_env_counts(bad)


def test_unknown_env_rejected():
    with pytest.raises(SystemExit):
        cli.make_parser().parse_args(["bench", "--env", "cartpole-xl"])


def test_constant_experience_horizons():
    """horizon = max(1, base * n_min // n) (reference cli.py:124-125)."""
    counts = [1024, 4096, 16384]
    n_min = min(counts)
    assert [max(1, (256 * n_min) // n) for n in counts] == [256, 64, 16]
