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


def validate_config(cfg, input_shape=None):
    """Spec checks and the shape chain (autobuild.py:73-113)."""
    if input_shape is None:
        input_shape = DATASET_SHAPES.get(cfg.train.dataset)
    for spec in cfg.layers:
        validate_spec(spec)
    if input_shape is None:
        return
    c, h, w = input_shape
    spatial, feat = (h, w), c
    for i, spec in enumerate(cfg.layers):
        if spec.kind == "fc":
            if spatial is not None:
                feat = feat * spatial[0] * spatial[1]
                spatial = None
            if spec.in_dim != feat:
                raise ConfigError(f"layer {i} expects in={spec.in_dim} but receives {feat} "
                                  f"features from layer {i - 1}")
        else:
            if spatial is None:
                raise ConfigError(f"layer {i}: conv after flattened features")
            if spec.in_dim != feat:
                raise ConfigError(f"layer {i} expects in={spec.in_dim} channels but layer "
                                  f"{i - 1} provides {feat}")
            if spec.kernel > spatial[0] + 2 * spec.pad or spec.kernel > spatial[1] + 2 * spec.pad:
                raise ConfigError(f"layer {i}: kernel {spec.kernel} larger than padded input {spatial}")
            spatial = output_spatial(spec, spatial)
        feat = spec.out_dim
    if spatial is not None:
        feat = feat * spatial[0] * spatial[1]
    if cfg.head.in_dim != feat:
        raise ConfigError(f"head expects in={cfg.head.in_dim} but receives {feat} features")


_LAYER_KEYS = ("family", "in", "out", "k", "s", "p", "bn", "act")
_TRAIN_KEYS = ("epochs", "batch", "lr", "seed", "dataset")


def _split_kv(parts, allowed, lineno):
    kv = {}
    for part in parts:
        if "=" not in part:
            raise ParseError(f"expected key=value, got {part!r}", lineno)
        key, value = part.split("=", 1)
        if key not in allowed:
            raise ParseError(f"unknown key {key!r}", lineno)
        if key in kv:
            raise ParseError(f"duplicate key {key!r}", lineno)
        kv[key] = value
    missing = [k for k in allowed if k not in kv]
    if missing:
        raise ParseError(f"missing keys {missing}", lineno)
    return kv


def _int(value, key, lineno):
    try:
        return int(value)
    except ValueError:
        raise ParseError(f"{key} must be an integer, got {value!r}", lineno) from None


def parse_config(text):
    """Config text -> ModelConfig; ParseError carries the line number."""
    name = head = train = None
    layers = []
    for lineno, raw in enumerate(text.splitlines(), start=1):
        line = raw.strip()
        if not line or line.startswith("#"):
            continue
        parts = line.split()
        word = parts[0]
        if word == "model":
            if name is not None:
                raise ParseError("duplicate model line", lineno)
            if len(parts) != 2:
                raise ParseError("model line must be 'model <name>'", lineno)
            name = parts[1]
        elif word == "layer":
            if len(parts) < 2 or parts[1] not in KINDS:
                raise ParseError(f"layer kind must be one of {KINDS}", lineno)
            if head is not None:
                raise ParseError("layer line after head", lineno)
            kv = _split_kv(parts[2:], _LAYER_KEYS, lineno)
            if kv["family"] not in FAMILIES or kv["family"] == "t2_linear":
                raise ParseError(f"unknown family tag {kv['family']!r}", lineno)
            if kv["act"] not in ("none", "relu"):
                raise ParseError(f"unknown activation {kv['act']!r}", lineno)
            if kv["bn"] not in ("0", "1"):
                raise ParseError(f"bn must be 0 or 1, got {kv['bn']!r}", lineno)
            spec = QuadraticLayerSpec(kind=parts[1], family=kv["family"], in_dim=_int(kv["in"], "in", lineno),
                                      out_dim=_int(kv["out"], "out", lineno), kernel=_int(kv["k"], "k", lineno),
                                      stride=_int(kv["s"], "s", lineno), pad=_int(kv["p"], "p", lineno),
                                      batchnorm=kv["bn"] == "1", activation=kv["act"])
            try:
                validate_spec(spec)
            except ConfigError as e:
                raise ParseError(str(e), lineno) from None
            layers.append(spec)
        elif word == "head":
            if head is not None:
                raise ParseError("duplicate head line", lineno)
            if len(parts) < 2 or parts[1] != "fc":
                raise ParseError("head must be 'head fc in=<n> classes=<k>'", lineno)
            kv = _split_kv(parts[2:], ("in", "classes"), lineno)
            head = HeadSpec(_int(kv["in"], "in", lineno), _int(kv["classes"], "classes", lineno))
        elif word == "train":
            if train is not None:
                raise ParseError("duplicate train line", lineno)
            kv = _split_kv(parts[1:], _TRAIN_KEYS, lineno)
            if kv["dataset"] not in DATASET_SHAPES:
                raise ParseError(f"dataset must be one of {sorted(DATASET_SHAPES)}", lineno)
            try:
                lr = float(kv["lr"])
            except ValueError:
                raise ParseError(f"lr must be a float, got {kv['lr']!r}", lineno) from None
            if not math.isfinite(lr) or lr <= 0:
                raise ParseError("lr must be positive and finite", lineno)
            train = TrainSpec(epochs=_int(kv["epochs"], "epochs", lineno), batch=_int(kv["batch"], "batch", lineno),
                              lr=lr, seed=_int(kv["seed"], "seed", lineno), dataset=kv["dataset"])
        else:
            raise ParseError(f"unknown directive {word!r}", lineno)
    if name is None:
        raise ParseError("missing model line")
    if head is None:
        raise ParseError("missing head line")
    if train is None:
        raise ParseError("missing train line")
    cfg = ModelConfig(name=name, layers=tuple(layers), head=head, train=train)
    validate_config(cfg)
    return cfg


def serialize_config(cfg):
    """Canonical text (byte-stable; parse(serialize(c)) == c)."""
    lines = [f"model {cfg.name}"]
    for spec in cfg.layers:
        lines.append("layer " + spec.describe())
    lines.append(f"head fc in={cfg.head.in_dim} classes={cfg.head.classes}")
    t = cfg.train
    lines.append(f"train epochs={t.epochs} batch={t.batch} lr={repr(float(t.lr))} seed={t.seed} "
                 f"dataset={t.dataset}")
    return "\n".join(lines) + "\n"


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


def save_checkpoint(model, path):
    """<path> (blob) + <path>.json (manifest), model.py:236-263. Returns the manifest."""
    entries = []
    blob = bytearray()
    records = [(tag, role, t) for tag, role, t in model.param_items()]
    for layer in model.layers:
        if isinstance(layer.core, QuadConvBN):
            records.append((layer.tag, "running_mean", layer.core.bn.running_mean))
            records.append((layer.tag, "running_var", layer.core.bn.running_var))
    for tag, role, t in records:
        raw = np.ascontiguousarray(t.detach().cpu().double().numpy(), dtype="<f8").tobytes()
        entries.append({"layer": tag, "role": role, "shape": list(t.shape), "offset": len(blob) + 8,
                        "length": len(raw)})
        blob.extend(struct.pack("<Q", len(raw)))
        blob.extend(raw)
    manifest = {"format": "quadra-checkpoint-v1", "config": serialize_config(model.cfg), "tensors": entries,
                "blob_sha256": hashlib.sha256(bytes(blob)).hexdigest(), "blob_bytes": len(blob)}
    with open(path, "wb") as f:
        f.write(bytes(blob))
    with open(str(path) + ".json", "w", encoding="utf-8") as f:
        json.dump(manifest, f, indent=1)
    return manifest


def load_checkpoint(path, compute_dtype=torch.float32, device=None):
    """Rebuild a QuadraModel from a checkpoint (model.py:266-300), verifying the manifest."""
    try:
        with open(str(path) + ".json", "r", encoding="utf-8") as f:
            manifest = json.load(f)
        with open(path, "rb") as f:
            blob = f.read()
    except OSError as e:
        raise IntegrityError(f"cannot read checkpoint {path}: {e}") from e
    if manifest.get("format") != "quadra-checkpoint-v1":
        raise IntegrityError(f"unknown checkpoint format in {path}.json")
    if len(blob) != manifest["blob_bytes"] or hashlib.sha256(blob).hexdigest() != manifest["blob_sha256"]:
        raise IntegrityError(f"checkpoint blob {path} does not match its manifest")
    cfg = parse_config(manifest["config"])
    model = QuadraModel(cfg, compute_dtype=compute_dtype, device=device)
    for entry in manifest["tensors"]:
        off, length = entry["offset"], entry["length"]
        (declared,) = struct.unpack("<Q", blob[off - 8:off])
        if declared != length:
            raise IntegrityError(f"length prefix {declared} != manifest length {length} at offset {off}")
        arr = np.frombuffer(blob[off:off + length], dtype="<f8").reshape(entry["shape"])
        model.set_param(entry["layer"], entry["role"], arr)
    return model
