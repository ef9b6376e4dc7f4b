"""Config text and checkpoint interop with the reference.

tests/golden/ckpt_tiny{,.json} were written by the REFERENCE's save_checkpoint
(oracle/gen_golden.py); ckpt_tiny_io.npz holds the reference's eval-mode logits.
CPU: config parse/serialise round trip and errors, checkpoint integrity checks,
load of the reference file, and a save whose manifest table matches the
reference's. GPU: the loaded model's logits on the B200 kernels.
"""
import hashlib
import json
import os
import struct

import numpy as np
import pytest
import torch

from conftest import GOLDEN
from oracle import quadra_oracle as Q
from paper_2204_01701_b200 import errors as E
from paper_2204_01701_b200 import model as M

CKPT = os.path.join(GOLDEN, "ckpt_tiny")


def _ref_manifest():
    with open(CKPT + ".json") as fh:
        return json.load(fh)


def test_config_roundtrip_matches_reference_serialisation():
    io = np.load(os.path.join(GOLDEN, "ckpt_tiny_io.npz"))
    text = str(io["serialized"])
    cfg = M.parse_config(text)
    assert M.serialize_config(cfg) == text
    assert M.parse_config(M.serialize_config(cfg)) == cfg
    assert _ref_manifest()["config"] == text


@pytest.mark.parametrize("text,line,msg", [
    ("model a\nmodel b\n", 2, "duplicate model line"),
    ("model a\nlayer bad family=t4\n", 2, "layer kind must be one of"),
    ("model a\nlayer fc family=zz in=1 out=1 k=1 s=1 p=0 bn=0 act=none\n", 2, "unknown family tag"),
    ("model a\nlayer fc family=t4 in=1 out=1 k=1 s=1 p=0 bn=2 act=none\n", 2, "bn must be 0 or 1"),
    ("model a\nlayer fc family=t4 in=1 out=1 k=3 s=1 p=0 bn=0 act=none\n", 2, "fc layers must use"),
    ("model a\nhead fc in=3 classes=2\ntrain epochs=1 batch=1 lr=-1 seed=0 dataset=mnist\n", 3, "lr must be"),
    ("model a\nfoo\n", 2, "unknown directive"),
])
def test_config_parse_errors(text, line, msg):
    with pytest.raises(E.ParseError, match=msg) as ei:
        M.parse_config(text)
    assert ei.value.line == line


def test_load_reference_checkpoint_and_resave_same_layout(tmp_path):
    mdl = M.load_checkpoint(CKPT)
    ref = _ref_manifest()
    with open(CKPT, "rb") as fh:
        blob = fh.read()
    # every tensor landed (fp32 masters: the reference's fp64 values, rounded)
    for e in ref["tensors"]:
        arr = np.frombuffer(blob[e["offset"]:e["offset"] + e["length"]], dtype="<f8").reshape(e["shape"])
        layer = mdl._by_tag(e["layer"])
        if e["role"] in ("gamma", "beta", "running_mean", "running_var"):
            t = {"gamma": layer.core.weight, "beta": layer.core.bias, "running_mean": layer.core.bn.running_mean,
                 "running_var": layer.core.bn.running_var}[e["role"]]
        else:
            t = getattr(layer.quad, e["role"])
        assert np.array_equal(t.detach().numpy(), arr.astype(np.float32)), (e["layer"], e["role"])
    # our writer: same (layer, role, shape, offset, length) table, valid digest
    out = tmp_path / "ck"
    man = M.save_checkpoint(mdl, out)
    assert [(t["layer"], t["role"], t["shape"], t["offset"], t["length"]) for t in man["tensors"]] == \
        [(t["layer"], t["role"], t["shape"], t["offset"], t["length"]) for t in ref["tensors"]]
    data = out.read_bytes()
    assert hashlib.sha256(data).hexdigest() == man["blob_sha256"] and len(data) == man["blob_bytes"]
    assert man["config"] == ref["config"] and man["format"] == "quadra-checkpoint-v1"
    # and it loads back to the same parameters
    m2 = M.load_checkpoint(out)
    for (t1, r1, a), (t2, r2, b) in zip(mdl.param_items(), m2.param_items()):
        assert (t1, r1) == (t2, r2) and torch.equal(a, b)


def test_checkpoint_integrity_errors(tmp_path):
    data = bytearray(open(CKPT, "rb").read())
    man = _ref_manifest()
    p = tmp_path / "bad"
    data[100] ^= 1  # corrupt one byte
    p.write_bytes(bytes(data))
    (tmp_path / "bad.json").write_text(json.dumps(man))
    with pytest.raises(E.IntegrityError, match="does not match its manifest"):
        M.load_checkpoint(p)
    man2 = dict(man, format="other")
    (tmp_path / "bad.json").write_text(json.dumps(man2))
    with pytest.raises(E.IntegrityError, match="unknown checkpoint format"):
        M.load_checkpoint(p)
    with pytest.raises(E.IntegrityError, match="cannot read"):
        M.load_checkpoint(tmp_path / "missing")
    # a wrong length prefix is caught even when the digest matches
    good = bytearray(open(CKPT, "rb").read())
    off = man["tensors"][0]["offset"]
    good[off - 8:off] = struct.pack("<Q", man["tensors"][0]["length"] + 8)
    man3 = dict(man, blob_sha256=hashlib.sha256(bytes(good)).hexdigest())
    p.write_bytes(bytes(good))
    (tmp_path / "bad.json").write_text(json.dumps(man3))
    with pytest.raises(E.IntegrityError, match="length prefix"):
        M.load_checkpoint(p)


@pytest.mark.gpu
def test_reference_checkpoint_logits_on_device():
    io = np.load(os.path.join(GOLDEN, "ckpt_tiny_io.npz"))
    mdl = M.load_checkpoint(CKPT, device="cuda").cuda().eval()
    x = torch.as_tensor(io["x"], dtype=torch.float32, device="cuda").contiguous(memory_format=torch.channels_last)
    with torch.no_grad():
        logits = mdl(x)
    assert Q.rel_err(logits.double().cpu().numpy(), io["logits"]) <= 1e-4
