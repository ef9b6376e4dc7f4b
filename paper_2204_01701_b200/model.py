"""Chain models from the reference's config files, and its checkpoint format
(checkpoint interop).

* Config text (reference autobuild.py:1-12, parse :153-228, serialize :235-245):
  ``model <name>`` / ``layer <kind> family=.. in=.. out=.. k=.. s=.. p=.. bn=0|1
  act=none|relu`` / ``head fc in=.. classes=..`` / ``train epochs=.. batch=..
  lr=.. seed=.. dataset=mnist|cifar10``; canonical serialisation is byte-stable.
* ``QuadraModel``: the reference Model (model.py:35-190) as torch modules on the
  B200 kernels -- body layers tagged ``L0, L1, ...`` (quadratic layer, optional
  batch norm with the reference semantics, optional ReLU, implicit flatten in
  front of an fc layer), then a first-order fc head tagged ``head``; parameters
  initialised with the reference draws (rng = default_rng((seed, i)), head
  (seed, 10000)).
* Checkpoints (model.py:236-300): a blob of little-endian float64 tensors, each
  prefixed by its u64 byte length, plus ``<path>.json`` with the config, the
  (layer, role, shape, offset, length) table and the blob's SHA-256. Files
  written here load in the reference and vice versa (tests/golden holds a
  reference-written checkpoint).
"""

from __future__ import annotations

import hashlib
import json
import math
import struct
from dataclasses import dataclass

import numpy as np
import torch
from torch import nn

from . import neurons
from .bn import QuadConvBN
from .errors import ConfigError, InputError, IntegrityError, ParseError
from .nn import _QuadBase
from .spec import FAMILIES, KINDS, QuadraticLayerSpec, output_spatial, validate_spec

DATASET_SHAPES = {"mnist": (1, 28, 28), "cifar10": (3, 32, 32)}
BN_EPS = 1e-5
BN_MOMENTUM = 0.1


@dataclass(frozen=True)
class HeadSpec:
    in_dim: int
    classes: int


@dataclass(frozen=True)
class TrainSpec:
    epochs: int
    batch: int
    lr: float
    seed: int
    dataset: str


@dataclass(frozen=True)
class ModelConfig:
    name: str
    layers: tuple
    head: HeadSpec
    train: TrainSpec


# ---------------------------------------------------------------------------
# config text: a small line grammar. Each directive names its fields; a field
# is (key, converter); the reader walks the lines once, the writer prints the
# same fields in the same order, so the text round-trips byte for byte.
# ---------------------------------------------------------------------------
def _as_int(key):
    def conv(v):
        try:
            return int(v)
        except ValueError:
            raise ValueError(f"{key} must be an integer, got {v!r}") from None
    return conv


def _one_of(key, choices, what):
    def conv(v):
        if v not in choices:
            raise ValueError(what.format(v=v))
        return v
    return conv


def _positive_float(v):
    try:
        f = float(v)
    except ValueError:
        raise ValueError(f"lr must be a float, got {v!r}") from None
    if not (math.isfinite(f) and f > 0):
        raise ValueError("lr must be positive and finite")
    return f


_LAYER_FIELDS = (("family", _one_of("family", tuple(f for f in FAMILIES if f != "t2_linear"),
                                    "unknown family tag {v!r}")),
                 ("in", _as_int("in")), ("out", _as_int("out")), ("k", _as_int("k")), ("s", _as_int("s")),
                 ("p", _as_int("p")), ("bn", _one_of("bn", ("0", "1"), "bn must be 0 or 1, got {v!r}")),
                 ("act", _one_of("act", ("none", "relu"), "unknown activation {v!r}")))
_HEAD_FIELDS = (("in", _as_int("in")), ("classes", _as_int("classes")))
_TRAIN_FIELDS = (("epochs", _as_int("epochs")), ("batch", _as_int("batch")), ("lr", _positive_float),
                 ("seed", _as_int("seed")),
                 ("dataset", _one_of("dataset", tuple(DATASET_SHAPES), f"dataset must be one of "
                                                                      f"{sorted(DATASET_SHAPES)}")))


def _read_fields(tokens, fields, lineno):
    """key=value tokens -> {key: converted value}; every field exactly once."""
    raw = {}
    names = [k for k, _ in fields]
    for tok in tokens:
        key, eq, value = tok.partition("=")
        if not eq:
            raise ParseError(f"expected key=value, got {tok!r}", lineno)
        if key not in names:
            raise ParseError(f"unknown key {key!r}", lineno)
        if key in raw:
            raise ParseError(f"duplicate key {key!r}", lineno)
        raw[key] = value
    absent = [k for k in names if k not in raw]
    if absent:
        raise ParseError(f"missing keys {absent}", lineno)
    out = {}
    for key, conv in fields:
        try:
            out[key] = conv(raw[key])
        except ValueError as e:
            raise ParseError(str(e), lineno) from None
    return out


class _ConfigReader:
    """Line-by-line state: at most one model / head / train line, layers before the head."""

    def __init__(self):
        self.name = self.head = self.train = None
        self.layers = []

    def _once(self, attr, lineno, word):
        if getattr(self, attr) is not None:
            raise ParseError(f"duplicate {word} line", lineno)

    def model(self, args, lineno):
        self._once("name", lineno, "model")
        if len(args) != 1:
            raise ParseError("model line must be 'model <name>'", lineno)
        self.name = args[0]

    def layer(self, args, lineno):
        if not args or args[0] not in KINDS:
            raise ParseError(f"layer kind must be one of {KINDS}", lineno)
        if self.head is not None:
            raise ParseError("layer line after head", lineno)
        f = _read_fields(args[1:], _LAYER_FIELDS, lineno)
        spec = QuadraticLayerSpec(kind=args[0], family=f["family"], in_dim=f["in"], out_dim=f["out"],
                                  kernel=f["k"], stride=f["s"], pad=f["p"], batchnorm=f["bn"] == "1",
                                  activation=f["act"])
        try:
            validate_spec(spec)
        except ConfigError as e:
            raise ParseError(str(e), lineno) from None
        self.layers.append(spec)

    def head_(self, args, lineno):
        self._once("head", lineno, "head")
        if not args or args[0] != "fc":
            raise ParseError("head must be 'head fc in=<n> classes=<k>'", lineno)
        f = _read_fields(args[1:], _HEAD_FIELDS, lineno)
        self.head = HeadSpec(f["in"], f["classes"])

    def train_(self, args, lineno):
        self._once("train", lineno, "train")
        f = _read_fields(args, _TRAIN_FIELDS, lineno)
        self.train = TrainSpec(epochs=f["epochs"], batch=f["batch"], lr=f["lr"], seed=f["seed"],
                               dataset=f["dataset"])

    def finish(self):
        for attr, word in (("name", "model"), ("head", "head"), ("train", "train")):
            if getattr(self, attr) is None:
                raise ParseError(f"missing {word} line")
        return ModelConfig(name=self.name, layers=tuple(self.layers), head=self.head, train=self.train)


def parse_config(text):
    """Config text -> ModelConfig (format of the reference autobuild.py:1-12);
    ParseError carries the 1-based line number."""
    rd = _ConfigReader()
    handlers = {"model": rd.model, "layer": rd.layer, "head": rd.head_, "train": rd.train_}
    for lineno, raw in enumerate(text.splitlines(), start=1):
        tokens = raw.split()
        if not tokens or tokens[0].startswith("#"):
            continue
        fn = handlers.get(tokens[0])
        if fn is None:
            raise ParseError(f"unknown directive {tokens[0]!r}", lineno)
        fn(tokens[1:], lineno)
    cfg = rd.finish()
    validate_config(cfg)
    return cfg


def serialize_config(cfg):
    """Canonical text: parse(serialize(c)) == c and serialize(parse(t)) == t for
    canonical t (the float lr printed with repr, as Python prints it)."""
    t = cfg.train
    rows = [("model", cfg.name)]
    rows += [("layer", spec.describe()) for spec in cfg.layers]
    rows.append(("head", f"fc in={cfg.head.in_dim} classes={cfg.head.classes}"))
    rows.append(("train", " ".join(f"{k}={v}" for k, v in (("epochs", t.epochs), ("batch", t.batch),
                                                          ("lr", repr(float(t.lr))), ("seed", t.seed),
                                                          ("dataset", t.dataset)))))
    return "".join(f"{word} {rest}\n" for word, rest in rows)


def _walk_shapes(cfg, input_shape):
    """Yield (index, spec, incoming (features, spatial or None)) along the chain,
    then ("head", None, (features, None)); fc layers flatten what they receive."""
    c, h, w = input_shape
    feat, spatial = c, (h, w)
    for i, spec in enumerate(cfg.layers):
        if spec.kind == "fc" and spatial is not None:
            feat, spatial = feat * spatial[0] * spatial[1], None
        yield i, spec, (feat, spatial)
        if spec.kind != "fc":
            spatial = output_spatial(spec, spatial) if spatial is not None else None
        feat = spec.out_dim
    if spatial is not None:
        feat = feat * spatial[0] * spatial[1]
    yield "head", None, (feat, None)


def validate_config(cfg, input_shape=None):
    """Every layer spec, then the shape chain (reference autobuild.py:73-113):
    channel / feature counts must meet, no conv after a flatten, kernels fit."""
    for spec in cfg.layers:
        validate_spec(spec)
    shape = input_shape if input_shape is not None else DATASET_SHAPES.get(cfg.train.dataset)
    if shape is None:
        return
    for i, spec, (feat, spatial) in _walk_shapes(cfg, shape):
        if i == "head":
            if cfg.head.in_dim != feat:
                raise ConfigError(f"head expects in={cfg.head.in_dim} but receives {feat} features")
        elif spec.kind == "fc":
            if spec.in_dim != feat:
                raise ConfigError(f"layer {i} expects in={spec.in_dim} but receives {feat} "
                                  f"features from layer {i - 1}")
        else:
            if spatial is None:
                raise ConfigError(f"layer {i}: conv after flattened features")
            if spec.in_dim != feat:
                raise ConfigError(f"layer {i} expects in={spec.in_dim} channels but layer "
                                  f"{i - 1} provides {feat}")
            if spec.kernel > min(spatial) + 2 * spec.pad:
                raise ConfigError(f"layer {i}: kernel {spec.kernel} larger than padded input {spatial}")


def _head_spec(head):
    return QuadraticLayerSpec(kind="fc", family="first_order", in_dim=head.in_dim, out_dim=head.classes)


class _Layer(nn.Module):
    """One body layer: quadratic layer [-> BN] [-> ReLU], implicit flatten before fc."""

    def __init__(self, spec, params, tag, compute_dtype, device):
        super().__init__()
        self.spec, self.tag = spec, tag
        q = _QuadBase(QuadraticLayerSpec(spec.kind, spec.family, spec.in_dim, spec.out_dim, spec.kernel,
                                         spec.stride, spec.pad), compute_dtype=compute_dtype, device=device)
        with torch.no_grad():
            for role, t in params.items():
                getattr(q, role).copy_(t)
        if spec.batchnorm:
            self.core = QuadConvBN(q, relu=spec.activation == "relu", momentum=BN_MOMENTUM, eps=BN_EPS)
            self.post_relu = False
        else:
            self.core = q
            self.post_relu = spec.activation == "relu"

    @property
    def quad(self):
        return self.core.layer if isinstance(self.core, QuadConvBN) else self.core

    def forward(self, x):
        if self.spec.kind == "fc" and x.dim() == 4:
            # NCHW flatten order (reference T.reshape of an NCHW array)
            x = x.contiguous().reshape(x.shape[0], -1)
        y = self.core(x)
        return torch.relu(y) if self.post_relu else y


class QuadraModel(nn.Module):
    """The reference chain model on the B200 kernels."""

    def __init__(self, cfg, compute_dtype=torch.float32, device=None, input_shape=None):
        super().__init__()
        validate_config(cfg, input_shape)
        self.cfg = cfg
        layers = []
        for i, spec in enumerate(cfg.layers):
            seed = spec.init_seed if spec.init_seed is not None else cfg.train.seed
            rng = np.random.default_rng((seed, i))
            params = neurons.init_params(spec, rng, device=device or "cpu")
            layers.append(_Layer(spec, params, f"L{i}", compute_dtype, device))
        hspec = _head_spec(cfg.head)
        rng = np.random.default_rng((cfg.train.seed, 10_000))
        layers.append(_Layer(hspec, neurons.init_params(hspec, rng, device=device or "cpu"), "head",
                             compute_dtype, device))
        self.layers = nn.ModuleList(layers)

    def forward(self, x):
        for layer in self.layers:
            x = layer(x)
        return x

    def _by_tag(self, tag):
        for layer in self.layers:
            if layer.tag == tag:
                return layer
        raise InputError(f"no layer tagged {tag!r}")

    def param_items(self):
        """(tag, role, tensor) in the reference walk order (model.py:67-76)."""
        out = []
        for layer in self.layers:
            q = layer.quad
            for role in sorted(neurons.param_shapes(q.spec)):
                out.append((layer.tag, role, getattr(q, role)))
            if isinstance(layer.core, QuadConvBN):
                out.append((layer.tag, "gamma", layer.core.weight))
                out.append((layer.tag, "beta", layer.core.bias))
        return out

    def set_param(self, tag, role, arr):
        layer = self._by_tag(tag)
        if role in ("gamma", "beta", "running_mean", "running_var"):
            if not isinstance(layer.core, QuadConvBN):
                raise IntegrityError(f"{tag} has no batch norm")
            t = {"gamma": layer.core.weight, "beta": layer.core.bias,
                 "running_mean": layer.core.bn.running_mean, "running_var": layer.core.bn.running_var}[role]
        else:
            t = getattr(layer.quad, role, None)
            if t is None:
                raise IntegrityError(f"{tag} has no parameter {role!r}")
        a = torch.as_tensor(np.array(arr, dtype=np.float64))  # owned copy (blob views are read-only)
        if tuple(a.shape) != tuple(t.shape):
            raise IntegrityError(f"{tag}/{role}: shape {tuple(a.shape)} != {tuple(t.shape)}")
        with torch.no_grad():
            t.copy_(a.to(t.dtype))


# ---------------------------------------------------------------------------
# checkpoints: quadra-checkpoint-v1 (reference model.py:236-300). The blob is
# a sequence of records, each a little-endian u64 byte count followed by that
# many bytes of little-endian float64 values; <path>.json holds the config
# text, one (layer, role, shape, offset, length) row per record (offset = the
# first value byte) and the blob's SHA-256 and size.
# ---------------------------------------------------------------------------
CKPT_FORMAT = "quadra-checkpoint-v1"
_U64 = struct.Struct("<Q")


class _BlobWriter:
    def __init__(self):
        self.buf = bytearray()
        self.rows = []

    def add(self, layer, role, values):
        data = np.ascontiguousarray(values, dtype="<f8")
        payload = data.tobytes()
        self.buf += _U64.pack(len(payload))
        self.rows.append({"layer": layer, "role": role, "shape": list(data.shape), "offset": len(self.buf),
                          "length": len(payload)})
        self.buf += payload

    def manifest(self, config_text):
        blob = bytes(self.buf)
        return blob, {"format": CKPT_FORMAT, "config": config_text, "tensors": self.rows,
                      "blob_sha256": hashlib.sha256(blob).hexdigest(), "blob_bytes": len(blob)}


class _BlobReader:
    def __init__(self, path):
        try:
            with open(str(path) + ".json", "r", encoding="utf-8") as fh:
                self.manifest = json.load(fh)
            with open(path, "rb") as fh:
                self.blob = fh.read()
        except OSError as e:
            raise IntegrityError(f"cannot read checkpoint {path}: {e}") from e
        m = self.manifest
        if m.get("format") != CKPT_FORMAT:
            raise IntegrityError(f"unknown checkpoint format in {path}.json")
        if len(self.blob) != m["blob_bytes"] or hashlib.sha256(self.blob).hexdigest() != m["blob_sha256"]:
            raise IntegrityError(f"checkpoint blob {path} does not match its manifest")

    def records(self):
        for row in self.manifest["tensors"]:
            off, n = row["offset"], row["length"]
            (prefix,) = _U64.unpack_from(self.blob, off - _U64.size)
            if prefix != n:
                raise IntegrityError(f"length prefix {prefix} != manifest length {n} at offset {off}")
            yield row["layer"], row["role"], np.frombuffer(self.blob, dtype="<f8", count=n // 8,
                                                           offset=off).reshape(row["shape"])


def _checkpoint_records(model):
    """(tag, role, tensor) in the reference's order: the parameter walk, then the
    BN running statistics layer by layer."""
    recs = list(model.param_items())
    for layer in model.layers:
        if isinstance(layer.core, QuadConvBN):
            recs += [(layer.tag, "running_mean", layer.core.bn.running_mean),
                     (layer.tag, "running_var", layer.core.bn.running_var)]
    return recs


def save_checkpoint(model, path):
    """Write <path> (blob) and <path>.json (manifest); returns the manifest."""
    w = _BlobWriter()
    for tag, role, t in _checkpoint_records(model):
        w.add(tag, role, t.detach().cpu().double().numpy())
    blob, manifest = w.manifest(serialize_config(model.cfg))
    with open(path, "wb") as fh:
        fh.write(blob)
    with open(str(path) + ".json", "w", encoding="utf-8") as fh:
        json.dump(manifest, fh, indent=1)
    return manifest


def load_checkpoint(path, compute_dtype=torch.float32, device=None):
    """A QuadraModel rebuilt from a verified checkpoint (digest, size, prefixes)."""
    rd = _BlobReader(path)
    model = QuadraModel(parse_config(rd.manifest["config"]), compute_dtype=compute_dtype, device=device)
    for tag, role, values in rd.records():
        model.set_param(tag, role, values)
    return model
