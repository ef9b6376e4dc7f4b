"""Layer specification, neuron-type tags and the integer shape/count logic.

This is the drop-in half of the boundary that never touches the GPU:

* :class:`QuadraticLayerSpec` has the reference's fields, order and defaults
  (/root/reference/pkg/src/quadra/autobuild.py:26-42).
* ``FAMILIES`` / ``KINDS`` / ``QUADRATIC_FAMILIES`` / ``T1_FAMILIES`` are the
  reference's tags (/root/reference/pkg/src/quadra/neurons.py:40-44) plus one
  new family, ``t2_linear`` = ``Wa (x*x) + Wc x`` (the north star's
  squared-input variant, which the reference does not define).
* ``validate_spec``, ``param_shapes``, ``cache_names``, ``count_*`` and
  ``conv_out_size`` reproduce neurons.py:50-186 and tensor.py:279-280 bit for
  bit (checked against golden vectors generated from the reference,
  tests/golden/spec_golden.json).

``DEVICE_FAMILIES`` / ``DEVICE_KINDS`` name what the sm_100a kernels
implement; ``validate_spec`` accepts every reference family (so configs parse
exactly as before) and the device entry points raise ``ConfigError`` for the
rest.
"""

from __future__ import annotations

from dataclasses import dataclass
from math import prod

from .errors import ConfigError, DimensionError

FAMILIES = ("first_order", "t1_pure", "t1_full", "t1and2",
            "t2", "t3", "t4", "t2and4", "proposed", "t2_linear")
QUADRATIC_FAMILIES = FAMILIES[1:]
T1_FAMILIES = ("t1_pure", "t1_full", "t1and2")
KINDS = ("fc", "conv", "dwconv")

# what the B200 kernels implement (the BASELINE.json hot path + first_order,
# which the degeneration tests compare against)
DEVICE_FAMILIES = ("first_order", "t1_pure", "t1_full", "t1and2", "t2", "t3", "t4", "t2and4", "proposed",
                   "t2_linear")
DEVICE_KINDS = ("fc", "conv", "dwconv")

# second factor of a product branch starts small (neurons.py:47, :142-143)
_DAMPED_SECOND_FACTOR = ("t4", "t2and4", "proposed")


@dataclass(frozen=True)
class QuadraticLayerSpec:
    """Reference autobuild.py:26-42, field for field."""
    kind: str
    family: str
    in_dim: int
    out_dim: int
    kernel: int = 1
    stride: int = 1
    pad: int = 0
    batchnorm: bool = False
    activation: str = "none"
    init_seed: int | None = None

    def describe(self):
        return (f"{self.kind} family={self.family} in={self.in_dim} "
                f"out={self.out_dim} k={self.kernel} s={self.stride} "
                f"p={self.pad} bn={int(self.batchnorm)} act={self.activation}")


def conv_out_size(size, r, stride, pad):
    """Floor-division output size (reference tensor.py:279-280)."""
    return (size + 2 * pad - r) // stride + 1


def validate_spec(spec):
    """Raise ConfigError if a layer spec is inconsistent (neurons.py:50-77).

    Messages match the reference text; tests/test_neurons.py:324-338 match on
    "fc", "single output" and "in == out".
    """
    if spec.family not in FAMILIES:
        raise ConfigError(f"unknown family {spec.family!r}")
    if spec.kind not in KINDS:
        raise ConfigError(f"unknown layer kind {spec.kind!r}")
    if spec.in_dim < 1 or spec.out_dim < 1:
        raise ConfigError(f"layer dims must be positive: {spec.in_dim}->{spec.out_dim}")
    if spec.family in T1_FAMILIES:
        if spec.kind != "fc":
            raise ConfigError(
                f"{spec.family} carries a full-rank quadratic weight and is "
                f"restricted to fc layers (got kind={spec.kind})")
        if spec.out_dim != 1:
            raise ConfigError(
                f"{spec.family} defines a single output unit; got out={spec.out_dim}")
    if spec.kind == "fc":
        if (spec.kernel, spec.stride, spec.pad) != (1, 1, 0):
            raise ConfigError("fc layers must use k=1 s=1 p=0")
    else:
        if spec.kernel < 1 or spec.stride < 1 or spec.pad < 0:
            raise ConfigError(
                f"bad conv geometry k={spec.kernel} s={spec.stride} p={spec.pad}")
    if spec.kind == "dwconv" and spec.in_dim != spec.out_dim:
        raise ConfigError(
            f"dwconv requires in == out channels, got {spec.in_dim}->{spec.out_dim}")
    if spec.activation not in ("none", "relu"):
        raise ConfigError(f"unknown activation {spec.activation!r}")


def validate_device_spec(spec):
    """validate_spec plus the subset the sm_100a kernels implement."""
    validate_spec(spec)
    if spec.family not in DEVICE_FAMILIES:
        raise ConfigError(
            f"family {spec.family!r} has no B200 kernel (supported: "
            f"{', '.join(DEVICE_FAMILIES)})")
    if spec.kind not in DEVICE_KINDS:
        raise ConfigError(
            f"kind {spec.kind!r} has no B200 kernel (supported: fc, conv, dwconv)")


def param_shapes(spec):
    """Role -> shape (neurons.py:80-107). fc weights are (in, out)."""
    validate_spec(spec)
    n, m, r = spec.in_dim, spec.out_dim, spec.kernel
    if spec.kind == "fc":
        w = (n, m)
    elif spec.kind == "conv":
        w = (m, n, r, r)
    else:
        w = (n, r, r)
    fam = spec.family
    if fam == "first_order":
        return {"W": w, "b": (m,)}
    if fam == "t1_pure":
        return {"Wq": (n, n)}
    if fam in ("t1_full", "t1and2"):
        return {"Wq": (n, n), "Wb": (n, 1)}
    if fam in ("t2", "t3"):
        return {"Wa": w}
    if fam == "t4":
        return {"Wa": w, "Wb": w}
    if fam == "t2and4":
        return {"Wa": w, "Wb": w, "Wc": w}
    if fam == "t2_linear":
        return {"Wa": w, "Wc": w}
    return {"Wa": w, "Wb": w, "Wc": w, "ba": (m,), "bb": (m,), "bc": (m,)}


def cache_names(family):
    """Minimal retained forward values (neurons.py:110-111)."""
    return ("x", "a", "b") if family in ("t4", "t2and4", "proposed") else ("x",)


def count_params(spec):
    return sum(int(prod(s)) for s in param_shapes(spec).values())


def count_weights(spec):
    """Parameter count excluding bias vectors (neurons.py:118-121)."""
    return sum(int(prod(s)) for role, s in param_shapes(spec).items()
               if not role.startswith("b"))


def fan_in(spec):
    if spec.kind == "fc":
        return spec.in_dim
    if spec.kind == "conv":
        return spec.in_dim * spec.kernel ** 2
    return spec.kernel ** 2


def count_macs(spec, input_shape=None):
    """Per-sample multiply count (neurons.py:150-186); (C, H, W) for conv."""
    validate_spec(spec)
    n, m = spec.in_dim, spec.out_dim
    fam = spec.family
    if spec.kind == "fc":
        lin = n * m
        sq_in, sq_out = n, m
    else:
        if input_shape is None or len(input_shape) != 3:
            raise DimensionError("conv MAC count needs an input shape (C, H, W)")
        c, h, w = input_shape
        if c != n:
            raise DimensionError(f"input channels {c} do not match spec in={n}")
        oh = conv_out_size(h, spec.kernel, spec.stride, spec.pad)
        ow = conv_out_size(w, spec.kernel, spec.stride, spec.pad)
        k2 = spec.kernel ** 2
        lin = (m * n * k2 if spec.kind == "conv" else n * k2) * oh * ow
        sq_in = c * h * w
        sq_out = m * oh * ow
    if fam == "first_order":
        return lin
    if fam == "t1_pure":
        return n * n + n
    if fam == "t1_full":
        return n * n + n + n
    if fam == "t1and2":
        return n + n * n + n + n
    if fam == "t2":
        return sq_in + lin
    if fam == "t3":
        return lin + sq_out
    if fam == "t4":
        return 2 * lin + sq_out
    if fam == "t2and4":
        return 3 * lin + sq_out + sq_in
    if fam == "t2_linear":
        return sq_in + 2 * lin
    return 3 * lin + sq_out


def output_spatial(spec, hw):
    h, w = hw
    if spec.kind == "fc":
        raise DimensionError("fc layers have no spatial size")
    return (conv_out_size(h, spec.kernel, spec.stride, spec.pad),
            conv_out_size(w, spec.kernel, spec.stride, spec.pad))


def gemm_branches(family):
    """Number of weight sets sharing the x operand in one fused GEMM.

    proposed: [Wa;Wb;Wc] -> 3; t4: [Wa;Wb] -> 2; t2/first_order: 1;
    t2_linear: 1 branch whose K is doubled ([x*x | x] against [Wa | Wc]).
    """
    return {"proposed": 3, "t4": 2, "t2": 1, "t3": 1, "first_order": 1, "t2_linear": 1, "t2and4": 3}[family]


def gemm_flops(spec, n, h=1, w=1):
    """Algorithmic fwd+bwd FLOPs (2*MAC of fprop + dgrad + wgrad GEMMs).

    Matches SURVEY.md §8(d): 3+3+3 GEMMs for proposed, 2+2+2 for t4 and
    t2_linear, 1+1+1 for t2/first_order; t2and4 3+3+3 (a, b on x, c on x*x);
    t3 1 + (1 recompute + 1 + 1) = 4 (the reference recomputes Wa x in the
    backward, neurons.py:406-411); elementwise work excluded.
    """
    if spec.kind == "fc":
        oh = ow = 1
        k = spec.in_dim
    else:
        oh = conv_out_size(h, spec.kernel, spec.stride, spec.pad)
        ow = conv_out_size(w, spec.kernel, spec.stride, spec.pad)
        k = spec.in_dim * spec.kernel ** 2
    one = 2 * n * oh * ow * k * spec.out_dim
    if spec.family in T1_FAMILIES:  # x Wq (n x n), x^T dv, dv Wq^T, + the recompute of x Wq
        return 4 * 2 * n * spec.in_dim * spec.in_dim
    if spec.kind == "dwconv":  # one r*r filter per channel
        one = 2 * n * oh * ow * spec.kernel ** 2 * spec.out_dim
    if spec.family == "t3":
        return 4 * one
    nb = {"proposed": 3, "t4": 2, "t2": 1, "first_order": 1, "t2_linear": 2, "t2and4": 3}[spec.family]
    return 3 * nb * one
