"""Host-side logic of config C2 (no GPU): the ResNet-50 program's geometry
and split-K / block sizing rules, the SGD segment table layout, the MMPP
trace helper and the bounded CPU-reference sample used by bench.py."""

import json
import math
import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

torch = pytest.importorskip("torch")

from paper_2410_07381_b200 import resnet  # noqa: E402


def test_resnet50_conv_geometry():
    """Stem 7x7/2 on 224 -> 112, maxpool -> 56; ResNet-50 v1.5 stride on the
    3x3 conv; K padded to 64 (the 8-channel stem: 7*7*8 = 392 -> 448)."""
    st = resnet.ConvSpec("conv1", resnet.IN_CH, 64, 7, 2, 3, 224, 224)
    assert (st.oh, st.ow, st.kdim, st.kp) == (112, 112, 392, 448)
    c2 = resnet.ConvSpec("layer2.0.conv2", 128, 128, 3, 2, 1, 56, 56)
    assert (c2.oh, c2.kdim, c2.kp, c2.direct) == (28, 1152, 1152, False)
    c1 = resnet.ConvSpec("layer1.0.conv1", 64, 64, 1, 1, 0, 56, 56)
    assert c1.direct and c1.kp == 64
    ds = resnet.ConvSpec("layer2.0.downsample.0", 256, 512, 1, 2, 0, 56, 56)
    assert not ds.direct and ds.oh == 28


@pytest.mark.parametrize("M,N,K", [(64, 448, 802816), (512, 4608, 3136), (200704, 576, 64), (3136, 512, 4608),
                                   (1024, 2048, 64), (12544, 256, 2304), (64, 64, 200704), (8, 2048, 1024)])
def test_gemm_splits_never_empty(M, N, K):
    S = resnet._gemm_splits(M, N, K)
    kb = math.ceil(K / 64)
    per = math.ceil(kb / S)
    assert 1 <= S <= max(1, kb)
    assert math.ceil(kb / per) == S          # every split has work (bind_gemm rejects empty splits)
    tiles = math.ceil(M / 128) * (N // (128 if N % 128 == 0 else 64))
    flops_per_block = 2.0 * 128 * (128 if N % 128 == 0 else 64) * per * 64
    assert S == 1 or flops_per_block <= 80e6 or S == kb // 2


@pytest.mark.parametrize("M,N,K", [(64, 576, 200704), (64, 448, 802816), (64, 256, 200704), (64, 64, 802816)])
def test_gemm_splits_bound_bytes_for_half_empty_tiles(M, N, K):
    """Weight gradients of 64-channel layers (M = 64 < 128: half-empty,
    memory-bound tiles) get <= ~256 KB of operands per logical block."""
    S = resnet._gemm_splits(M, N, K)
    kb = math.ceil(K / 64)
    per = math.ceil(kb / S)
    bn = 128 if N % 128 == 0 else 64
    assert math.ceil(kb / per) == S
    assert per * 2 * (M + bn) * 64 <= 262144


def test_bn_rows_per_block():
    assert resnet._rb(802816, 64) == 1024 and resnet._rb(802816, 64, 4) == 256
    assert resnet._rb(3136, 2048) == 80 and resnet._rb(3136, 2048, 4) == 64
    assert resnet._rb(3136, 512) == 32


def test_sgd_table_layout():
    """96-byte nn::SgdSeg records (incl. the flipped conv-weight copy) and a
    (segment, chunk) map covering every element (kernels_nn.cu SgdUpdate);
    segments with many gradient partials get smaller logical blocks."""
    import numpy as np
    w = torch.zeros(96, 200)
    v = torch.zeros_like(w)
    g = torch.zeros(3, 96, 200)
    w2 = torch.zeros(5000)
    t = resnet.SgdTable()
    t.add(w, v, g, 3, 96 * 200, 1e-4, rows=96, cols=200)
    t.add(w2, torch.zeros_like(w2), torch.zeros(1, 5000), 1, 5000, 0.0)
    t.build("cpu")
    raw = t.dev_segs.numpy().view(np.uint8)
    assert raw.size == 2 * 96
    rec = np.frombuffer(raw.tobytes(), dtype=np.dtype({
        "names": ["w", "n", "gstride", "S", "rows", "cols", "chunk", "wf", "fk"],
        "formats": ["<u8", "<i8", "<i8", "<i4", "<i4", "<i4", "<i4", "<u8", "<i4"],
        "offsets": [0, 24, 32, 40, 64, 68, 72, 80, 88], "itemsize": 96}))
    assert rec["wf"][0] == 0 and rec["fk"][0] == 0
    assert rec["w"][0] == w.data_ptr() and rec["n"][0] == 19200 and rec["S"][0] == 3
    assert rec["gstride"][1] == 5000 and rec["rows"][0] == 96 and rec["cols"][0] == 200
    m = t.dev_map.numpy()
    assert rec["chunk"][0] == 1024 and rec["chunk"][1] == 1024
    assert t.blocks == math.ceil(19200 / 1024) + math.ceil(5000 / 1024) == len(m)
    many = resnet.SgdTable()
    many.add(torch.zeros(4096), torch.zeros(4096), torch.zeros(64, 4096), 64, 4096, 0.0)
    many.build("cpu")
    assert many.blocks == 4096 // 128
    assert sorted(set(m[:, 0].tolist())) == [0, 1]
    with pytest.raises(ValueError):
        bad = resnet.SgdTable()
        bad.add(torch.zeros(6), torch.zeros(6), torch.zeros(1, 6), 1, 6, 0.0)
        bad.build("cpu")


def test_c2_trace_is_deterministic_and_loaded():
    import bench
    hp_ns = 850_000
    a = bench.c2_trace(0.25, hp_ns, int(20e9), 3, 4.0)
    assert a == bench.c2_trace(0.25, hp_ns, int(20e9), 3, 4.0)
    assert all(x < 20e9 for x in a) and list(a) == sorted(a)
    load = len(a) * hp_ns / 20e9
    assert 0.12 < load < 0.45      # MMPP: mean load 0.25, bursty


def test_cpu_reference_models_every_kernel():
    """The CPU reference arm models every best-effort kernel of the step (not
    a prefix) and the HP request, from the committed B200-measured costs."""
    import bench
    for cfg in ("c2", "c3", "c4"):
        costs = json.load(open(os.path.join(ROOT, "profiles", f"{cfg}_costs.json")))
        hp, be = bench.ref_tasks(costs)
        assert len(be) == len(costs["be"]) and len(hp) >= 1
        assert all(w.cost.total_blocks == k["blocks"] for w, k in zip(be, costs["be"]))
        assert all(w.exempt for w in hp)


@pytest.mark.parametrize("M,N,K", [(4096, 1024, 4096), (4096, 3072, 1024), (1024, 4096, 4096), (30720, 1024, 4096),
                                   (4096, 1024, 30720), (4096, 512, 64), (256, 256, 64), (4096, 4096, 100)])
def test_pair_plan_never_empty(M, N, K):
    """CTA-pair plans: pair tiles only for N % 256 == 0 and >= 32 tiles, no
    empty split, pair logical blocks <= ~180 MFLOP unless K is too short to split."""
    import math
    from paper_2410_07381_b200.transformer import _pair_plan
    pair, S = _pair_plan(M, N, K)
    kb = math.ceil(K / 64)
    per = math.ceil(kb / S)
    assert 1 <= S <= max(1, kb) and math.ceil(kb / per) == S
    if pair:
        assert N % 256 == 0 and math.ceil(M / 256) * (N // 256) >= 32
        assert 2 * 256 * 256 * per * 64 <= 200e6 or per <= 2
    assert not _pair_plan(M, N, K, enabled=False)[0]
