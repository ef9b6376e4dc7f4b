"""Integer shape/count logic of the product (paper_2204_01701_b200.spec) is
bit-exact against golden vectors produced by the reference itself."""
import json
import os

import pytest

from conftest import GOLDEN
from paper_2204_01701_b200 import errors as E
from paper_2204_01701_b200 import spec as S

with open(os.path.join(GOLDEN, "spec_golden.json")) as fh:
    G = json.load(fh)


def test_validate_and_shapes_match_reference():
    n_ok = 0
    for row in G["specs"]:
        sp = S.QuadraticLayerSpec(**row["spec"])
        if not row["ok"]:
            with pytest.raises(E.ConfigError) as ei:
                S.validate_spec(sp)
            assert row["error"] == "ConfigError"
            assert str(ei.value) == row["message"]
            continue
        n_ok += 1
        S.validate_spec(sp)
        assert sp.describe() == row["describe"]
        assert {k: list(v) for k, v in S.param_shapes(sp).items()} == row["param_shapes"]
        assert S.count_params(sp) == row["count_params"]
        assert S.count_weights(sp) == row["count_weights"]
        assert list(S.cache_names(sp.family)) == row["cache_names"]
        if sp.kind == "fc":
            assert S.count_macs(sp) == row["count_macs"]
        else:
            for hw, want in row["count_macs"].items():
                h, w = map(int, hw.split("x"))
                if isinstance(want, str):
                    with pytest.raises(getattr(E, want)):
                        S.count_macs(sp, (sp.in_dim, h, w))
                else:
                    assert S.count_macs(sp, (sp.in_dim, h, w)) == want
    assert n_ok > 100


def test_conv_out_size_bit_exact():
    for size, r, s, p, want in G["conv_out_size"]:
        assert S.conv_out_size(size, r, s, p) == want


def test_error_messages_match_reference_regexes():
    # reference tests/test_neurons.py:324-338
    with pytest.raises(E.ConfigError, match="fc"):
        S.validate_spec(S.QuadraticLayerSpec(kind="conv", family="t1_pure", in_dim=3, out_dim=1,
                                             kernel=3))
    with pytest.raises(E.ConfigError, match="single output"):
        S.validate_spec(S.QuadraticLayerSpec(kind="fc", family="t1_full", in_dim=3, out_dim=2))
    with pytest.raises(E.ConfigError, match="in == out"):
        S.validate_spec(S.QuadraticLayerSpec(kind="dwconv", family="t4", in_dim=3, out_dim=4,
                                             kernel=3))


def test_device_spec_gate():
    S.validate_device_spec(S.QuadraticLayerSpec(kind="conv", family="proposed", in_dim=64,
                                                out_dim=64, kernel=3, pad=1))
    S.validate_device_spec(S.QuadraticLayerSpec(kind="fc", family="t3", in_dim=4, out_dim=4))
    S.validate_device_spec(S.QuadraticLayerSpec(kind="conv", family="t2and4", in_dim=4, out_dim=4,
                                                kernel=3, pad=1))
    S.validate_device_spec(S.QuadraticLayerSpec(kind="fc", family="t1_pure", in_dim=4, out_dim=1))
    with pytest.raises(E.ConfigError, match="single output"):
        S.validate_device_spec(S.QuadraticLayerSpec(kind="fc", family="t1_pure", in_dim=4,
                                                    out_dim=2))
    with pytest.raises(E.ConfigError, match="fc layers"):
        S.validate_device_spec(S.QuadraticLayerSpec(kind="conv", family="t1_full", in_dim=4,
                                                    out_dim=1, kernel=3))
    S.validate_device_spec(S.QuadraticLayerSpec(kind="dwconv", family="t4", in_dim=4,
                                                out_dim=4, kernel=3))
    with pytest.raises(E.ConfigError, match="in == out"):
        S.validate_device_spec(S.QuadraticLayerSpec(kind="dwconv", family="t4", in_dim=4,
                                                    out_dim=8, kernel=3))


def test_t2_linear_counters():
    sp = S.QuadraticLayerSpec(kind="conv", family="t2_linear", in_dim=3, out_dim=6, kernel=3,
                              pad=1)
    assert S.param_shapes(sp) == {"Wa": (6, 3, 3, 3), "Wc": (6, 3, 3, 3)}
    lin = 6 * 3 * 9 * 8 * 8
    assert S.count_macs(sp, (3, 8, 8)) == 3 * 8 * 8 + 2 * lin
    assert S.cache_names("t2_linear") == ("x",)


def test_baseline_flop_counts():
    # C2 proposed fwd+bwd = 86.97 GFLOP; C1 = 1.208 GFLOP
    c2 = S.QuadraticLayerSpec(kind="conv", family="proposed", in_dim=64, out_dim=64, kernel=3,
                              pad=1)
    assert S.gemm_flops(c2, 128, 32, 32) == 9 * 2 * 131072 * 576 * 64
    c1 = S.QuadraticLayerSpec(kind="fc", family="proposed", in_dim=512, out_dim=512)
    assert S.gemm_flops(c1, 256) == 9 * 2 * 256 * 512 * 512
