"""Boundary types: PipelineConfig / GmmParams / PbasParams validation.

The rules are the reference's (GmmParams.validate gmm.py:53-62,
PbasParams.validate pbas.py:57-63, PipelineConfig.validate config.py:37-50);
the device-path limits (pbas.n <= 255, k <= 16) apply only to the algorithm
that runs, so any config the reference accepts for that algorithm passes.
"""

import pytest

from paper_2002_00250_b200.config import GmmParams, PbasParams, PipelineConfig, validate_config
from paper_2002_00250_b200.errors import ConfigError


def test_defaults_validate():
    PipelineConfig().validate()
    PipelineConfig(algorithm="pbas").validate()


@pytest.mark.parametrize("bad", [
    dict(algorithm="svm"), dict(mode="depth_only"), dict(workers=0), dict(seed=-1),
    dict(seed=2 ** 64), dict(gmm=GmmParams(k_rgb=0)), dict(gmm=GmmParams(tau=0.0)),
    dict(pbas=PbasParams(n=1, min_matches=2)), dict(pbas=PbasParams(t_init=1.0)),
    dict(pbas=PbasParams(r_lower=0.0)), dict(gmm_state_dtype="float16"),
])
def test_reference_rules_raise_config_error(bad):
    with pytest.raises(ConfigError):
        PipelineConfig(**bad).validate()


def test_device_limits_only_for_the_algorithm_that_runs():
    # pbas.n > 255 does not fit the u8 ring state; irrelevant for GMM
    validate_config(PipelineConfig(algorithm="gmm", pbas=PbasParams(n=300)))
    with pytest.raises(ConfigError, match="pbas.n"):
        validate_config(PipelineConfig(algorithm="pbas", pbas=PbasParams(n=300)))
    validate_config(PipelineConfig(algorithm="pbas", gmm=GmmParams(k_rgb=40)))
    with pytest.raises(ConfigError, match="k_rgb"):
        validate_config(PipelineConfig(algorithm="gmm", gmm=GmmParams(k_rgb=40)))


def test_duck_typed_config():
    class Cfg:
        algorithm, mode, seed, workers = "pbas", "rgb_only", 5, 2
        gmm, pbas = GmmParams(), PbasParams(n=7)

    validate_config(Cfg())
