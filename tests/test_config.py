"""Boundary types: the key=value config system (reference config.py:53-125)."""

import pytest

from paper_2002_00250_b200.config import (ConfigError, PipelineConfig, apply_param_overrides,
                                          default_workers, effective_config_lines,
                                          parse_config_file)
from paper_2002_00250_b200.errors import ConfigError as CE


def test_parse_config_file(tmp_path):
    p = tmp_path / "run.conf"
    p.write_text("# comment\n\nalgo = pbas\n gmm.tau =  2.5 \npbas.n=12\n")
    assert parse_config_file(p) == {"algo": "pbas", "gmm.tau": "2.5", "pbas.n": "12"}
    bad = tmp_path / "bad.conf"
    bad.write_text("algo pbas\n")
    with pytest.raises(CE, match="bad.conf:1: expected 'key = value'"):
        parse_config_file(bad)
    with pytest.raises(CE, match="not found"):
        parse_config_file(tmp_path / "missing.conf")


def test_apply_param_overrides_types_and_errors():
    cfg = PipelineConfig()
    apply_param_overrides(cfg, {"gmm.tau": "2.5", "pbas.n": "12", "gmm.k_rgb": "5"})
    assert cfg.gmm.tau == 2.5 and cfg.pbas.n == 12 and cfg.gmm.k_rgb == 5
    assert isinstance(cfg.pbas.n, int) and isinstance(cfg.gmm.tau, float)
    for bad in ({"tau": "1"}, {"gmm.nope": "1"}, {"svm.c": "1"}, {"pbas.n": "x"}):
        with pytest.raises(ConfigError):
            apply_param_overrides(PipelineConfig(), bad)


def test_default_workers(monkeypatch):
    monkeypatch.delenv("RGBD_BGSEG_WORKERS", raising=False)
    assert default_workers() == 1
    monkeypatch.setenv("RGBD_BGSEG_WORKERS", "6")
    assert default_workers() == 6
    for bad in ("0", "x"):
        monkeypatch.setenv("RGBD_BGSEG_WORKERS", bad)
        with pytest.raises(ConfigError):
            default_workers()


def test_effective_config_lines():
    lines = effective_config_lines(PipelineConfig(algorithm="pbas", seed=3), {"z": 1, "a": 2})
    assert lines[:4] == ["algo = pbas", "mode = rgbd", "seed = 3", "workers = 1"]
    assert "gmm.k_rgb = 7" in lines and "pbas.n = 20" in lines
    assert lines[-2:] == ["a = 2", "z = 1"]
