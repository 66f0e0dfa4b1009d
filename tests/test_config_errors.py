"""The reference's error contract on the host side (CPU, no GPU needed):
QuantConfig validation (reference tests/test_blockquant.py TestConfigValidation),
both error types being ValueError subclasses (errors.py), the ABI return
codes mapped onto them (_lib.check), and argument checks the package makes
before any launch."""

import numpy as np
import pytest

import paper_2512_02010_b200 as f46
from paper_2512_02010_b200 import _lib
from paper_2512_02010_b200.errors import ConfigError, InvalidInputError


def test_error_types_are_value_errors():
    assert issubclass(ConfigError, ValueError)
    assert issubclass(InvalidInputError, ValueError)


def test_adaptive_forces_cap_256():
    assert f46.QuantConfig(scale_mode="adaptive").fp8_cap == 256.0
    with pytest.raises(ConfigError):
        f46.QuantConfig(scale_mode="adaptive", fp8_cap=448.0)


def test_default_cap_448():
    assert f46.QuantConfig().fp8_cap == 448.0
    with pytest.raises(ConfigError):
        f46.QuantConfig(fp8_cap=300.0)


@pytest.mark.parametrize("kw", [dict(fmt="int4"), dict(scale_mode="fixed5"), dict(rule="mad"),
                                dict(rounding="up"), dict(seed=-1), dict(seed=1.5)])
def test_bad_enums_and_seeds(kw):
    with pytest.raises(ConfigError):
        f46.QuantConfig(**kw)


def test_mxfp4_rejects_non_fixed6():
    with pytest.raises(ConfigError):
        f46.QuantConfig(fmt="mxfp4", scale_mode="adaptive")
    with pytest.raises(ConfigError):
        f46.QuantConfig(fmt="mxfp4", scale_mode="fixed4")


@pytest.mark.parametrize("t", [6.5, -0.1])
def test_threshold_range(t):
    with pytest.raises(InvalidInputError):
        f46.QuantConfig(threshold=t)


@pytest.mark.parametrize("rc,exc", [(_lib.F46_ERR_INVALID_ARG, InvalidInputError),
                                    (_lib.F46_ERR_CONFIG, ConfigError),
                                    (_lib.F46_ERR_UNSUPPORTED, InvalidInputError),
                                    (_lib.F46_ERR_CUDA, RuntimeError)])
def test_abi_return_codes_map_to_reference_errors(rc, exc):
    with pytest.raises(exc):
        _lib.check(rc, "f46_test")
    _lib.check(_lib.F46_OK, "f46_test")


def test_block_api_argument_checks_precede_launch():
    # validation errors are raised before anything reaches the device
    with pytest.raises(InvalidInputError):
        f46.quantize_block(np.zeros((2, 2)), 1.0, 6.0)
    with pytest.raises(InvalidInputError):
        f46.quantize_block(np.array([]), 1.0, 6.0)
    with pytest.raises(InvalidInputError):
        f46.quantize_block(np.array([1.0, np.nan]), 1.0, 6.0)
    with pytest.raises(ConfigError):
        f46.quantize_block(np.ones(4), 1.0, 6.0, rounding="up")
    with pytest.raises(InvalidInputError):
        f46.quantize_block(np.ones(4), 1.0, 6.0, rounding="sr")
    with pytest.raises(InvalidInputError):
        f46.quantize_block(np.ones(4), 1.0, 6.0, rounding="sr", u=np.zeros(3))
    with pytest.raises(ConfigError):
        f46.quantize_block_adaptive(np.ones(4), 1.0, rule="mad")
    with pytest.raises(InvalidInputError):
        f46.quantize_block_adaptive(np.ones(4), 1.0, rounding="sr", u6=np.zeros(4))
    with pytest.raises(InvalidInputError):
        f46.compute_block_scale(np.ones(4), 0.0, 6.0)
    with pytest.raises(InvalidInputError):
        f46.compute_block_scale(np.ones(4), float("inf"), 6.0)
