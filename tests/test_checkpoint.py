"""SADDCKPT hand-off: the reference-written container
(tests/golden/toy_moe.saddckpt, made by tests/golden/make_golden.py with the
real reference's save_checkpoint) parses, re-serialises byte for byte, and
rejects malformed input like the reference (ref checkpoint.py:100-137,
docs/formats.md). The GPU tests build the device model from it and compare the
forward logits and `evaluate` dispatch maps with the reference's own."""

import os

import numpy as np
import pytest
import torch

from paper_2306_06446_b200 import checkpoint as CK

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
CKPT = os.path.join(GOLDEN, "toy_moe.saddckpt")


def test_load_reference_checkpoint():
    ck = CK.load_checkpoint(CKPT)
    assert ck.version == 1 and ck.step == 42 and ck.meta["note"] == "golden fixture"
    cfg = ck.model_config
    assert len(cfg.blocks) == 2 and cfg.blocks[0].mlp_mode == "moe" and cfg.img == 16
    assert ck.arrays["patch_embed.w"].shape == (48, 32)
    assert ck.arrays["block0.mlp.router.wg"].shape == (32, 2)
    assert ck.arrays["block1.mlp.fc1.quant_p"].dtype == np.int32
    assert ck.meta["quant"] == {"p_min": -15, "p_max": 15, "scale_mode": "per-matrix"}


def test_rewrite_is_byte_identical(tmp_path):
    ck = CK.load_checkpoint(CKPT)
    out = tmp_path / "re.saddckpt"
    CK.write_container(out, ck.meta, ck.arrays)
    assert out.read_bytes() == open(CKPT, "rb").read()


@pytest.mark.parametrize("cut", [0, 5, 11, 15, 40, 300, -7])
def test_truncations_raise_format_error(tmp_path, cut):
    data = open(CKPT, "rb").read()
    p = tmp_path / "t.saddckpt"
    p.write_bytes(data[:cut] if cut >= 0 else data[:len(data) + cut])
    with pytest.raises(CK.FormatError):
        CK.load_checkpoint(p)


def test_bad_magic_and_version(tmp_path):
    data = bytearray(open(CKPT, "rb").read())
    p = tmp_path / "m.saddckpt"
    bad = bytearray(data)
    bad[0:8] = b"NOTACKPT"
    p.write_bytes(bytes(bad))
    with pytest.raises(CK.FormatError, match="offset 0"):
        CK.load_checkpoint(p)
    bad = bytearray(data)
    bad[8:12] = (2).to_bytes(4, "little")
    p.write_bytes(bytes(bad))
    with pytest.raises(CK.VersionError):
        CK.load_checkpoint(p)


# ------------------------------------------------------------------ GPU


def _dataset(g):
    class DS:
        images = g["images"]
        labels = g["labels"]
    return DS()


@pytest.mark.gpu
def test_build_model_forward_matches_reference(golden):
    g = golden("checkpoint")
    m = CK.build_model(CK.load_checkpoint(CKPT))
    logits = m.forward(torch.from_numpy(g["images"]).cuda()).cpu().numpy()
    ref = g["logits"]
    assert np.max(np.abs(logits - ref)) / np.max(np.abs(ref)) < 1e-5


@pytest.mark.gpu
def test_evaluate_dispatch_maps_match_reference(golden, tmp_path):
    from paper_2306_06446_b200 import model as MD
    g = golden("checkpoint")
    m = CK.build_model(CK.load_checkpoint(CKPT))
    res = MD.evaluate(m, _dataset(g), batch_size=3)
    names = [k[4:] for k in g if k.startswith("map:")]
    assert sorted(res.dispatch_maps) == sorted(names)
    for name in names:
        assert np.array_equal(res.dispatch_maps[name], g["map:" + name]), name
        assert res.expert_shares[name] == list(g["share:" + name]), name
    assert res.accuracy == float(g["accuracy"])
    csv_path = MD.write_dispatch_map(res, "block0.mlp", tmp_path)
    rows = open(csv_path).read().splitlines()
    assert rows[0] == "image," + ",".join(f"token{t}" for t in range(16))
    assert rows[1] == "0," + ",".join(str(v) for v in g["map:block0.mlp"][0])
    import json
    summ = json.loads((tmp_path / "dispatch_summary.json").read_text())
    assert summ["tokens_per_image"] == 16 and summ["images"] == 5 and summ["layer"] == "block0.mlp"


@pytest.mark.gpu
def test_save_from_device_is_byte_identical(tmp_path):
    ck = CK.load_checkpoint(CKPT)
    m = CK.build_model(ck)
    out = tmp_path / "dev.saddckpt"
    CK.save_checkpoint(out, m, step=42, extra_meta={"note": "golden fixture"})
    assert out.read_bytes() == open(CKPT, "rb").read()


@pytest.mark.gpu
def test_build_model_rejects_bad_records():
    ck = CK.load_checkpoint(CKPT)
    missing = CK.Checkpoint(ck.version, ck.model_config,
                            {k: v for k, v in ck.arrays.items() if k != "head.w"}, ck.step, ck.meta)
    with pytest.raises(CK.FormatError, match="missing parameter 'head.w'"):
        CK.build_model(missing)
    arrays = dict(ck.arrays)
    arrays["pos"] = arrays["pos"][:-1]
    with pytest.raises(CK.FormatError, match="shape mismatch"):
        CK.build_model(CK.Checkpoint(ck.version, ck.model_config, arrays, ck.step, ck.meta))
    arrays = dict(ck.arrays)
    arrays["block1.mlp.fc1.quant_p"] = arrays["block1.mlp.fc1.quant_p"] + 1
    with pytest.raises(CK.FormatError, match="disagrees"):
        CK.build_model(CK.Checkpoint(ck.version, ck.model_config, arrays, ck.step, ck.meta))
