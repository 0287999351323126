"""Golden fixtures written by the UNMODIFIED reference (tests/golden/make_golden.py): they pin the
oracle and the "MOE1" file format where /root/reference does not exist (the GPU box)."""
import ctypes as C
import os

import numpy as np
import pytest

from oracle.pyoracle import Config, Oracle

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
MOE_PLAIN = os.path.join(GOLDEN, "moe1_e4k2d8n16_seed1.moe")
MOE_SHARED = os.path.join(GOLDEN, "moe1_e3k2d8n8s4_seed7.moe")


@pytest.fixture(scope="module")
def oracle():
    return Oracle.get()


@pytest.fixture(scope="module")
def skb():
    import paper_2605_08575_b200 as m
    return m


def golden_layer_case(oracle):
    cfg = Config(8, 2, 96, 160, 48, True)
    synth = oracle.generate_synthetic(cfg, 11, 0.1)
    w = synth.rounded_bf16()
    w.router = synth.router  # the device image keeps the router in fp32
    g = np.load(os.path.join(GOLDEN, "layer_e8k2d96n160s48.npz"))
    return cfg, w, g


def test_oracle_reproduces_the_reference_layer_outputs(oracle):
    cfg, w, g = golden_layer_case(oracle)
    x = g["x"]
    assert x.tobytes() == oracle.round_bf16(oracle.generate_tokens(5, cfg.d_model, 4)).tobytes()
    y, _ = oracle.forward(w, x)
    assert y.tobytes() == g["y_dense"].tobytes()
    routed, shared = oracle.build_topk_masks(w, x, 0.5, 1)
    np.testing.assert_array_equal(routed.reshape(-1), g["routed"].reshape(-1))
    np.testing.assert_array_equal(shared.reshape(-1), g["shared"].reshape(-1))
    y, rep = oracle.forward(w, x, g["routed"], g["shared"])
    assert y.tobytes() == g["y_masked"].tobytes()
    assert rep.active_neurons_total == int(g["rep_masked"][0])
    rc, y, rep = oracle.forward_sparse(w, x, 0.05)
    assert rc == 0 and y.tobytes() == g["y_sparse"].tobytes()
    got = [rep.gate_macs, rep.up_macs, rep.down_macs, rep.other_macs, rep.active_neurons_total,
           rep.tiles_total, rep.tiles_skipped]
    assert got == [int(v) for v in g["rep_sparse"]]


def _file_matrices(path, cfg):
    raw = np.fromfile(path, dtype="<f4", offset=28)
    E, N, D, S = cfg.n_experts, cfg.d_ffn, cfg.d_model, cfg.d_shared
    router, rest = raw[:E * D].reshape(E, D), raw[E * D:]
    experts = rest[:3 * E * N * D].reshape(E, 3, N, D)
    tail = rest[3 * E * N * D:]
    shared = tail.reshape(3, S, D) if S else None
    return router, experts, shared


@pytest.mark.parametrize("path,cfg,seed", [(MOE_PLAIN, Config(4, 2, 8, 16, 0, True), 1),
                                           (MOE_SHARED, Config(3, 2, 8, 8, 4, False), 7)])
def test_moe1_files_of_the_reference(oracle, skb, path, cfg, seed, tmp_path):
    """Layout (model.cpp:190-216), closed-form size (model.cpp:180-188), and our writer
    reproducing the reference's file byte for byte."""
    blob = open(path, "rb").read()
    scfg = skb.MoEConfig(cfg.n_experts, cfg.top_k, cfg.d_model, cfg.d_ffn, cfg.has_shared,
                         cfg.d_shared, cfg.renormalize, 64)
    assert len(blob) == skb.weight_file_size(scfg)
    assert blob[:4] == b"MOE1"
    hdr = np.frombuffer(blob[4:28], "<u4")
    assert list(hdr) == [cfg.n_experts, cfg.top_k, cfg.d_model, cfg.d_ffn, cfg.d_shared,
                         (1 if cfg.has_shared else 0) | (2 if cfg.renormalize else 0)]
    w = oracle.generate_synthetic(cfg, seed, 0.05)
    router, experts, shared = _file_matrices(path, cfg)
    assert router.tobytes() == w.router.tobytes()
    assert experts[:, 0].tobytes() == w.gate.tobytes() and experts[:, 1].tobytes() == w.up.tobytes()
    assert experts[:, 2].tobytes() == w.down_t.tobytes()
    if cfg.has_shared:
        assert shared[0].tobytes() == w.shared_gate.tobytes()
        assert shared[2].tobytes() == w.shared_down_t.tobytes()
    if seed == 1:  # proj/tests/golden/gen_e4k2d8n16_seed1_router_row0.txt
        assert [int(v) for v in router[0].view(np.uint32)][:3] == [0x3bda1bda, 0x3cc9582a, 0x3d40ec37]
    out = tmp_path / "ours.moe"
    skb.save_weights(scfg, out, w.router, w.gate, w.up, w.down_t, w.shared_gate, w.shared_up,
                     w.shared_down_t)
    assert open(out, "rb").read() == blob


def test_moe1_loader_format_errors(skb, tmp_path):
    """model_test.cpp:129-205: offsets of the reference's FormatError cases; every one of them is
    raised before the device is touched."""
    blob = bytearray(open(MOE_PLAIN, "rb").read())

    def load(data):
        p = tmp_path / "case.moe"
        p.write_bytes(bytes(data))
        return skb.MoELayerWeights.load(p)

    with pytest.raises(skb.FormatError) as e:
        load(b"XXXX" + bytes(64))
    assert e.value.offset == 0 and "bad magic, expected MOE1 (offset 0)" in str(e.value)
    keep = 28 + (4 * 8 + 3 * 16 * 8) * 4  # header, router, the first expert only
    with pytest.raises(skb.FormatError) as e:
        load(blob[:keep])
    assert e.value.offset >= keep - 4 and "truncated file" in str(e.value)
    with pytest.raises(skb.FormatError) as e:
        load(blob[:keep + 3])  # the reference reads whole words
    assert e.value.offset == keep
    with pytest.raises(skb.FormatError) as e:
        load(blob[:10])
    assert e.value.offset == 8
    bad = bytearray(blob)
    bad[8] = 77  # top_k low byte: K > E
    with pytest.raises(skb.FormatError) as e:
        load(bad)
    assert e.value.offset == 8
    for off, val in ((4, 0), (12, 0), (16, 0)):
        bad = bytearray(blob)
        bad[off:off + 4] = val.to_bytes(4, "little")
        with pytest.raises(skb.FormatError) as e:
            load(bad)
        assert e.value.offset == off
    bad = bytearray(blob)
    bad[24] |= 1  # shared flag without d_shared
    with pytest.raises(skb.FormatError) as e:
        load(bad)
    assert e.value.offset == 20
    with pytest.raises(skb.FormatError) as e:
        load(blob + b"\0")
    assert e.value.offset == len(blob) and "trailing bytes" in str(e.value)
    with pytest.raises(skb.IoError):
        skb.MoELayerWeights.load(tmp_path / "missing.moe")


def test_weight_file_size_does_not_wrap(skb):
    """Header fields are 31-bit values: 3*E*N*D*4 wraps 64 bits for a crafted header.  The size is
    formed in 128 bits and reported as 0 (no such file), so that the loader rejects the header
    before it builds pointers past the mapping."""
    big = skb.MoEConfig(2**31 - 1, 1, 2**31 - 1, 2**31 - 1, False, 0, True, 64)
    assert skb.weight_file_size(big) == 0
    ok = skb.MoEConfig(4, 2, 8, 16, False, 0, True, 64)
    assert skb.weight_file_size(ok) == 28 + 4 * 8 * 4 + 3 * 4 * 16 * 8 * 4


def test_report_file_is_the_reference_byte_for_byte(skb, ref, tmp_path):
    """emit_report / read_report (profiler.cpp:221-286): our writer against the reference's own on
    the same points, the parse back, and the FormatError offsets."""
    import numpy as np
    pts = np.array([[0.0, 0.0, 0.0, 1.0, 0.0],
                    [0.25, 0.249987654321, 0.25, 0.987654321987, 1.2345678912e-2],
                    [0.5, 0.5, 0.5, 1.0 / 3.0, 2.0 / 3.0],
                    [0.9, 0.8999999999, 0.9, 1e-12, 123456789.123]], np.float64)
    theirs = tmp_path / "ref.csv"
    assert ref.lib.ref_emit_report(pts, len(pts), b"R+S", 0.5, str(theirs).encode()) == 0
    res = skb.SweepResult([skb.SweepPoint(*row, path="R+S") for row in pts], 0.5)
    ours = tmp_path / "ours.csv"
    skb.emit_report(res, ours)
    assert ours.read_bytes() == theirs.read_bytes()
    back = skb.read_report(theirs)
    assert back.cutoff == 0.5 and len(back.points) == 4 and back.points[1].path == "R+S"
    assert back.points[2].quality == float("%.9g" % (1.0 / 3.0))
    empty = tmp_path / "empty.csv"
    skb.emit_report(skb.SweepResult(), empty)
    assert empty.read_text() == skb.REPORT_HEADER + "\n"   # no cutoff line without points
    bad = tmp_path / "bad.csv"
    bad.write_text("not the header\n")
    with pytest.raises(skb.FormatError) as e:
        skb.read_report(bad)
    assert e.value.offset == 0
    bad.write_text(skb.REPORT_HEADER + "\n0,0,0,1,0,R\n0.5,0.5\n")
    with pytest.raises(skb.FormatError) as e:
        skb.read_report(bad)
    assert e.value.offset == len(skb.REPORT_HEADER) + 1 + len("0,0,0,1,0,R") + 1
    with pytest.raises(skb.IoError):
        skb.read_report(tmp_path / "missing.csv")
