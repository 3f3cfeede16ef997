"""GPU: the weight-gradient GEMM on the tensor cores and the fused backward
sink.

* samo_dw_gemm_f16 vs the reference's matmul(transpose(x), dy)
  (train.hpp:304, tensor.hpp:88-105; the oracle's restatement equals it bit
  for bit, test_oracle.py).  The tensor cores add the exact products in a
  different order, so the tolerance per element is one binary16 ulp of the
  reference value plus 2*batch*2^-24*sum_b |x_b*dy_b| (fp32 summation-order
  bound).  Most elements come out identical.
* samo_model_sink_dw (GEMM with the gather in its epilogue) is bit-identical
  to the unfused path: dense dW from samo_dw_gemm_f16 -> samo_model_sink_dense
  (K1), and a whole step through it equals the set_grads + step path.
"""
from __future__ import annotations

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def S(cuda):
    from paper_2302_05045_b200 import samo
    return samo


def _half(rng, shape, scale):
    return torch.from_numpy((rng.uniform(-1, 1, shape) * scale).astype(np.float16)).cuda()


def _bits(t):
    return t.cpu().numpy().view(np.uint16)


def _ulp16(h_bits):
    f = np.abs(h_bits.view(np.float16).astype(np.float64))
    e = np.floor(np.log2(np.maximum(f, 2.0 ** -14)))
    return 2.0 ** (e - 10)


# batch <= 1024 runs the two-epilogue-group variant, larger batches the other
SHAPES = [(576, 128, 128), (64, 256, 384), (100, 136, 200), (1, 8, 8), (576, 1024, 512), (130, 8, 264),
          (1100, 256, 384), (2048, 512, 264),
          (130, 2560, 2560)]  # 100 pair tiles over 74 pairs: a partial second wave


_REF = {}  # (batch, in, out) -> (x, dy, reference bits, tolerance): the oracle GEMM runs once per shape


def _reference(oracle, batch, n_in, n_out):
    key = (batch, n_in, n_out)
    if key not in _REF:
        rng = np.random.default_rng(batch * 7 + n_in)
        x = _half(rng, (batch, n_in), 1.0)
        dy = _half(rng, (batch, n_out), 1024.0 / batch)  # loss-scaled softmax grads (train.hpp:276)
        xb, db = _bits(x), _bits(dy)
        want = oracle.dw_matmul(xb, db)
        absum = np.abs(xb.view(np.float16).astype(np.float64)).T @ np.abs(db.view(np.float16).astype(np.float64))
        _REF[key] = (x, dy, want, _ulp16(want) + 2.0 * batch * 2.0 ** -24 * absum)
    return _REF[key]


@pytest.mark.parametrize("batch,n_in,n_out", SHAPES)
def test_dw_gemm_vs_reference(S, oracle, batch, n_in, n_out):
    x, dy, want, tol = _reference(oracle, batch, n_in, n_out)
    got = _bits(S.dw_gemm(x, dy))
    gf = got.view(np.float16).astype(np.float64)
    wf = want.view(np.float16).astype(np.float64)
    bad = np.abs(gf - wf) > tol
    assert not bad.any(), (int(bad.sum()), np.argwhere(bad)[:5])
    assert np.mean(got == want) > 0.5


# Long-K shapes under each launch form (the launcher reads the knobs on every
# call): MS = 1 / 2 / 3 (256 x 256, 512 x 256 or 256 x 384 pair tiles), with
# and without the tail-wave split; ragged M (520: a partly out-of-range
# sub-tile) and N (8, 1032: out-of-range dY boxes in the 384-wide form).
FORMS = [{"SAMO_DW_MS": "1", "SAMO_DW_TAIL": "1"}, {"SAMO_DW_MS": "1", "SAMO_DW_TAIL": "0"},
         {"SAMO_DW_MS": "2"}, {"SAMO_DW_MS": "2", "SAMO_DW_MS2_EW": "1"},
         {"SAMO_DW_MS": "3"}, {"SAMO_DW_MS": "3", "SAMO_DW_W_EW": "1"},
         {"SAMO_DW_MS": "3", "SAMO_DW_W_EW": "2"}]  # 3: the 256 x 384 pair tile (3 epilogue groups by default)
LONG_K = [(1100, 256, 384), (1100, 520, 1032), (1100, 2560, 2560), (3000, 136, 8)]


@pytest.mark.parametrize("form", FORMS, ids=lambda f: "-".join(f"{k[8:]}{v}" for k, v in f.items()))
@pytest.mark.parametrize("batch,n_in,n_out", LONG_K)
def test_dw_gemm_forms_vs_reference(S, oracle, monkeypatch, form, batch, n_in, n_out):
    for k, v in form.items():
        monkeypatch.setenv(k, v)
    test_dw_gemm_vs_reference(S, oracle, batch, n_in, n_out)


@pytest.mark.parametrize("form", FORMS, ids=lambda f: "-".join(f"{k[8:]}{v}" for k, v in f.items()))
def test_sink_dw_forms_equal_unfused(S, monkeypatch, form):
    for k, v in form.items():
        monkeypatch.setenv(k, v)
    rng = np.random.default_rng(29)
    shapes = [(2560, 2560), (520, 1032)]
    fused, unfused = _model(S, shapes, 0.9, 10), _model(S, shapes, 0.9, 10)
    for l, (i, o) in enumerate(shapes):
        x, dy = _half(rng, (1100, i), 1.0), _half(rng, (1100, o), 2.0)
        fused.sink_dw(l, x, dy)
        unfused.sink_dense(l, S.dw_gemm(x, dy).reshape(-1))
    torch.cuda.synchronize()
    for l in range(len(shapes)):
        assert np.array_equal(_bits(fused.read(l, "grad16")), _bits(unfused.read(l, "grad16"))), l


def test_dw_gemm_errors(S):
    x = torch.zeros((4, 12), dtype=torch.float16, device="cuda")
    dy = torch.zeros((4, 16), dtype=torch.float16, device="cuda")
    with pytest.raises(S.DimensionError):
        S.dw_gemm(x, dy)  # in = 12 is not a multiple of 8
    with pytest.raises(S.DimensionError):
        S.dw_gemm(torch.zeros((4, 16), dtype=torch.float16, device="cuda"),
                  torch.zeros((5, 16), dtype=torch.float16, device="cuda"))


def _model(S, shapes, p, seed):
    rng = np.random.default_rng(seed)
    sets = []
    for l, (i, o) in enumerate(shapes):
        n = i * o
        keep = max(1, int(round((1 - p) * n)))
        idx = np.sort(rng.choice(n, size=keep, replace=False)).astype(np.uint32)
        sets.append(S.PrunedIndexSet(f"fc{l}.weight", n, torch.from_numpy(idx.view(np.int32)).cuda()))
    m = S.SamoModel.from_index_sets(sets, [tuple(s) for s in shapes], 0)
    for l, (i, o) in enumerate(shapes):
        m.init_layer(l, torch.from_numpy(rng.uniform(-0.05, 0.05, i * o).astype(np.float32)).cuda())
    m.set_config(S.OptimizerConfig(learning_rate=1e-2, loss_scale=1024.0))
    return m


FC = [(256, 384), (384, 136), (136, 64)]


@pytest.mark.parametrize("batch", [200, 1500])
def test_sink_dw_equals_unfused_gather(S, batch):
    rng = np.random.default_rng(5)
    fused, unfused = _model(S, FC, 0.9, 1), _model(S, FC, 0.9, 1)
    for l, (i, o) in enumerate(FC):
        x, dy = _half(rng, (batch, i), 1.0), _half(rng, (batch, o), 4.0)
        fused.sink_dw(l, x, dy)
        unfused.sink_dense(l, S.dw_gemm(x, dy).reshape(-1))
    torch.cuda.synchronize()
    for l in range(len(FC)):
        assert np.array_equal(_bits(fused.read(l, "grad16")), _bits(unfused.read(l, "grad16"))), l


def test_sink_dw_step_matches_dense_path(S):
    """Three steps: fused sinks + update == dense dW + set_grads + step."""
    rng = np.random.default_rng(9)
    batch = 96
    fused, dense = _model(S, FC, 0.8, 3), _model(S, FC, 0.8, 3)
    for s in range(3):
        ins = [(_half(rng, (batch, i), 1.0), _half(rng, (batch, o), 8.0)) for i, o in FC]
        for l in reversed(range(len(FC))):  # backward order
            fused.sink_dw(l, *ins[l])
        fused.update()
        dense.set_grads([S.dw_gemm(x, dy).reshape(-1) for x, dy in ins])
        dense.step()
    for l in range(len(FC)):
        for k in ("theta32", "adam_m", "adam_v"):
            assert np.array_equal(fused.read(l, k).cpu().numpy().view(np.uint32),
                                  dense.read(l, k).cpu().numpy().view(np.uint32)), (l, k)
        assert np.array_equal(_bits(fused.read(l, "theta16")), _bits(dense.read(l, "theta16")))
    a, b = fused.step_record(), dense.step_record()
    assert (a.t, a.skipped_steps) == (b.t, b.skipped_steps) == (3, 0)
    fused.check_invariants()


def test_sink_dw_nonfinite_skips(S):
    rng = np.random.default_rng(11)
    m = _model(S, FC, 0.9, 4)
    before = m.read(0, "theta32").clone()
    for l, (i, o) in enumerate(FC):
        x, dy = _half(rng, (64, i), 1.0), _half(rng, (64, o), 1.0)
        if l == 0:
            dy[:, :] = float("inf")  # every dW element of layer 0 is +-inf or NaN
        m.sink_dw(l, x, dy)
    m.update()
    r = m.step_record()
    assert (r.t, r.skipped_steps) == (0, 1)
    assert torch.equal(before, m.read(0, "theta32"))


def test_sink_errors(S):
    m = _model(S, FC, 0.9, 6)
    x = torch.zeros((8, 256), dtype=torch.float16, device="cuda")
    with pytest.raises(S.DimensionError):
        m.sink_dw(0, x, torch.zeros((8, 136), dtype=torch.float16, device="cuda"))  # 256 x 136 != 256 x 384
    with pytest.raises(S.SamoIndexError):
        m.sink_dw(7, x, torch.zeros((8, 384), dtype=torch.float16, device="cuda"))


@pytest.mark.parametrize("shapes,p", [([(8, 8), (24, 16)], 0.0),        # every element kept
                                      ([(16, 8), (8, 264)], 0.9999),    # one kept element per layer
                                      ([(136, 72)], 0.5)])
def test_sink_dw_density_edges(S, shapes, p):
    rng = np.random.default_rng(17)
    batch = 33
    fused, unfused = _model(S, shapes, p, 8), _model(S, shapes, p, 8)
    for l, (i, o) in enumerate(shapes):
        x, dy = _half(rng, (batch, i), 1.0), _half(rng, (batch, o), 2.0)
        fused.sink_dw(l, x, dy)
        unfused.sink_dense(l, S.dw_gemm(x, dy).reshape(-1))
    torch.cuda.synchronize()
    for l in range(len(shapes)):
        assert np.array_equal(_bits(fused.read(l, "grad16")), _bits(unfused.read(l, "grad16"))), l


def test_sink_dw_many_tiles_equals_unfused(S):
    """2560 x 2560 (100 pair tiles over 74 pairs, a partial second wave): the
    fused sink still equals dense dW -> K1."""
    rng = np.random.default_rng(23)
    shapes = [(2560, 2560)]
    fused, unfused = _model(S, shapes, 0.9, 9), _model(S, shapes, 0.9, 9)
    for batch in (300, 1500):  # both epilogue variants
        x, dy = _half(rng, (batch, 2560), 1.0), _half(rng, (batch, 2560), 2.0)
        fused.sink_dw(0, x, dy)
        unfused.sink_dense(0, S.dw_gemm(x, dy).reshape(-1))
        torch.cuda.synchronize()
        assert np.array_equal(_bits(fused.read(0, "grad16")), _bits(unfused.read(0, "grad16"))), batch

