"""DLRM with TT fields on the GPU vs the unmodified reference's DlrmModel
(golden run in tests/golden/dlrm.npz: fp32 model, 3 SGD+momentum steps)."""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def test_dlrm_matches_reference_run(golden):
    from paper_2507_14668_b200.model import DlrmModel, ModelConfig, bags_field_tensors
    torch.backends.cuda.matmul.allow_tf32 = False
    s = golden("dlrm")
    cfg = ModelConfig(n_dense=6, rows_per_field=(4000, 500, 118), emb_dim=16, ranks=(1, 4, 4, 1), tt_threshold=1000,
                      bottom_sizes=(32,), top_sizes=(32, 16), loss="bce", seed=5)
    model = DlrmModel(cfg)
    params = dict(model.named_ref_params())
    # initialisation: same seeded stream, same order -> identical bits
    for name, p in params.items():
        assert np.array_equal(p.detach().cpu().numpy(), s[f"init.{name}"]), name
    dense = torch.from_numpy(s["data.dense"].astype(np.float32)).cuda()
    labels = torch.from_numpy(s["data.labels"]).cuda()
    bs = 32
    for step in range(3):
        lo, hi = step * bs, (step + 1) * bs
        sparse = []
        for f in range(3):
            idx, off = s[f"data.idx{f}"], s[f"data.off{f}"]
            sub_idx = idx[off[lo]:off[hi]]
            sub_off = off[lo:hi + 1] - off[lo]
            sparse.append((torch.from_numpy(sub_idx).cuda(), torch.from_numpy(sub_off).cuda()))
        loss = model.train_step(dense[lo:hi], sparse, labels[lo:hi], lr=0.05, momentum=0.9)
        assert abs(loss - s["losses"][step]) <= 1e-5 * max(1.0, abs(s["losses"][step])), (step, loss)
        for name, p in params.items():
            got = p.detach().cpu().numpy().astype(np.float64)
            want = s[f"step{step}.{name}"].astype(np.float64)
            err = np.abs(got - want).max() / max(1e-3, np.abs(want).max())
            assert err < 1e-4, (step, name, err)


def test_checkpoint_bytes_match_reference(golden, tmp_path):
    """TTCKPT1 of the freshly initialised model == the reference's bytes;
    save -> load round trip restores every parameter; corrupt files raise."""
    from paper_2507_14668_b200 import model as M
    s = golden("dlrm")
    cfg = M.ModelConfig(n_dense=6, rows_per_field=(4000, 500, 118), emb_dim=16, ranks=(1, 4, 4, 1),
                        tt_threshold=1000, bottom_sizes=(32,), top_sizes=(32, 16), loss="bce", seed=5)
    model = M.DlrmModel(cfg)
    assert M.checkpoint_bytes(model) == s["ckpt_init"].tobytes()
    # the reference's post-training checkpoint loads here with the same tensors
    path = tmp_path / "ref.ckpt"
    path.write_bytes(s["ckpt_final"].tobytes())
    loaded = M.load_checkpoint(path)
    for name, p in loaded.named_ref_params():
        assert np.array_equal(p.detach().cpu().numpy(), s[f"step2.{name}"]), name
    assert M.checkpoint_bytes(loaded) == s["ckpt_final"].tobytes()
    M.save_checkpoint(loaded, tmp_path / "mine.ckpt")
    assert (tmp_path / "mine.ckpt").read_bytes() == s["ckpt_final"].tobytes()
    # corruption
    bad = tmp_path / "bad.ckpt"
    bad.write_bytes(b"NOTCKPT" + s["ckpt_final"].tobytes()[7:])
    with pytest.raises(ValueError):
        M.load_checkpoint(bad)
    bad.write_bytes(s["ckpt_final"].tobytes()[:-3])
    with pytest.raises(ValueError):
        M.load_checkpoint(bad)


def test_dlrm_tensor_core_pipeline_matches_reference(golden):
    """The same reference train_step (model.py:347-365) with the production
    TT geometry (emb 64, ranks (1, 32, 32, 1)), so the TT field runs the
    tensor-core pipeline (k_fplan / k_fwd / k_bwd / fused SGD) — golden run in
    tests/golden/dlrm_tc.npz (make_golden.py gen_dlrm_tc)."""
    from paper_2507_14668_b200.embedding_bag import TTEmbeddingBag
    from paper_2507_14668_b200.model import DlrmModel, ModelConfig
    torch.backends.cuda.matmul.allow_tf32 = False
    s = golden("dlrm_tc")
    rows = (12000, 700)
    cfg = ModelConfig(n_dense=5, rows_per_field=rows, emb_dim=64, ranks=(1, 32, 32, 1), tt_threshold=1000,
                      bottom_sizes=(32,), top_sizes=(32,), loss="bce", seed=9)
    model = DlrmModel(cfg)
    assert isinstance(model.fields[0], TTEmbeddingBag) and model.fields[0].engine.fast
    params = dict(model.named_ref_params())
    for name, p in params.items():
        assert np.array_equal(p.detach().cpu().numpy(), s[f"init.{name}"]), name
    dense = torch.from_numpy(s["data.dense"].astype(np.float32)).cuda()
    labels = torch.from_numpy(s["data.labels"]).cuda()
    bs = 64
    for step in range(3):
        lo, hi = step * bs, (step + 1) * bs
        sparse = []
        for f in range(len(rows)):
            idx, off = s[f"data.idx{f}"], s[f"data.off{f}"]
            sparse.append((torch.from_numpy(idx[off[lo]:off[hi]]).cuda(),
                           torch.from_numpy(off[lo:hi + 1] - off[lo]).cuda()))
        loss = model.train_step(dense[lo:hi], sparse, labels[lo:hi], lr=0.05, momentum=0.9)
        assert abs(loss - s["losses"][step]) <= 1e-5 * max(1.0, abs(s["losses"][step])), (step, loss)
        for name, p in params.items():
            got = p.detach().cpu().numpy().astype(np.float64)
            want = s[f"step{step}.{name}"].astype(np.float64)
            err = np.abs(got - want).max() / max(1e-3, np.abs(want).max())
            assert err < 1e-4, (step, name, err)


def test_dlrm_batched_tt_fields_match_per_field():
    """DlrmModel serves its TT fields from ONE table-batched collection
    (batch_tt_fields, §8 f1) with the per-field model's exact initial
    parameters (the reference's init order) and training trajectory (three
    SGD + momentum steps: losses and every parameter within fp32 noise)."""
    import numpy as np
    import torch
    from paper_2507_14668_b200.model import DlrmModel, ModelConfig, checkpoint_bytes
    cfg = ModelConfig(n_dense=5, rows_per_field=(12000, 700, 30000, 4000), emb_dim=64, ranks=(1, 32, 32, 1),
                      tt_threshold=1000, bottom_sizes=(32,), top_sizes=(32,), loss="bce", seed=9)
    a = DlrmModel(cfg, batch_size=128)
    b = DlrmModel(cfg, batch_tt_fields=False)
    assert a.tt is not None and a.tt.num_tables == 3 and b.tt is None
    assert checkpoint_bytes(a) == checkpoint_bytes(b)
    rng = np.random.default_rng(4)
    torch.backends.cuda.matmul.allow_tf32 = False
    for step in range(3):
        B = 128
        dense = torch.from_numpy(rng.standard_normal((B, 5)).astype(np.float32)).cuda()
        labels = torch.from_numpy((rng.random(B) < 0.3).astype(np.float64)).cuda()
        sparse = []
        for rows in cfg.rows_per_field:
            sizes = rng.integers(1, 4, size=B)
            idx = rng.integers(0, rows, size=int(sizes.sum()))
            off = np.concatenate([[0], np.cumsum(sizes)])
            sparse.append((torch.from_numpy(idx).cuda(), torch.from_numpy(off).cuda()))
        la = a.train_step(dense, sparse, labels, 0.05, 0.9)
        lb = b.train_step(dense, sparse, labels, 0.05, 0.9)
        assert abs(la - lb) <= 1e-6 * max(1.0, abs(lb)), step
    for (na, pa), (nb, pb) in zip(a.named_ref_params(), b.named_ref_params()):
        assert na == nb
        d = (pa.detach() - pb.detach()).abs().max().item()
        assert d <= 1e-5 * max(1e-3, pb.detach().abs().max().item()), na
