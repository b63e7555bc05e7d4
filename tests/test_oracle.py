"""CPU checks of the numerics oracle and the TP shard bookkeeping (no GPU).

* oracle/gpt_oracle.py's Philox-4x32-10 is pinned by the published Random123 known-answer
  vectors (kat_vectors: philox4x32_10 with zero, all-ones and pi-digit counters / keys);
* the dropout keep-mask it derives keeps a fraction 1 - p and is a pure function of
  (seed, stream, element);
* the Megatron shard map the device initialiser uses (ops_elementwise.cu
  init_normal_sharded_kernel) and executor.unshard are inverse to each other.
"""
import numpy as np
import pytest

from oracle import gpt_oracle as go

KAT = [
    ((0, 0, 0, 0), (0, 0), (0x6627E8D5, 0xE169C58D, 0xBC57AC4C, 0x9B00DBD8)),
    ((0xFFFFFFFF,) * 4, (0xFFFFFFFF, 0xFFFFFFFF), (0x408F276D, 0x41C83B0E, 0xA20BC7C6, 0x6D5451FD)),
    ((0x243F6A88, 0x85A308D3, 0x13198A2E, 0x03707344), (0xA4093822, 0x299F31D0),
     (0xD16CFE09, 0x94FDCCEB, 0x5001E420, 0x24126EA1)),
]


@pytest.mark.parametrize("ctr,key,want", KAT)
def test_philox_known_answers(ctr, key, want):
    out = go.philox4x32_10(tuple(np.array([c], dtype=np.uint64) for c in ctr), key)
    assert tuple(int(x[0]) for x in out) == want


def test_keep_mask_rate_and_purity():
    m = go.keep_mask(go.step_seed(42, 1), go.layer_stream(3, 1, go.SITE_ATTN), 1 << 18, 0.1)
    assert abs(m.mean() - 0.9) < 0.003
    # prefix property: element e depends only on (seed, stream, e)
    assert np.array_equal(go.keep_mask(go.step_seed(42, 1), go.layer_stream(3, 1, go.SITE_ATTN), 1000, 0.1), m[:1000])
    other = go.keep_mask(go.step_seed(42, 1), go.layer_stream(3, 2, go.SITE_ATTN), 1 << 18, 0.1)
    assert (m != other).mean() > 0.1
    assert go.keep_mask(1, 2, 100, 0.0).all()
    assert go.drop_threshold(0.1) == int(float(np.float32(0.1)) * 2**16) == 6553


def _shard(full: np.ndarray, base: str, tp: int, r: int) -> np.ndarray:
    """numpy restatement of init_normal_sharded_kernel's index map (rows, cols, row_blk, col_split)."""
    h = full.shape[1] if full.ndim == 2 and base in ("w_qkv", "w_fc1") else full.shape[0]
    if base in ("w_proj", "w_fc2"):
        cols = full.shape[1] // tp
        return full[:, r * cols:(r + 1) * cols]
    blk = {"w_qkv": h // tp, "b_qkv": full.shape[0] // 3 // tp, "w_fc1": full.shape[0] // tp,
           "b_fc1": full.shape[0] // tp}[base]
    rows = full.shape[0] // tp
    idx = [(i // blk) * blk * tp + r * blk + i % blk for i in range(rows)]
    return full[idx]


@pytest.mark.parametrize("tp", [1, 2, 4])
@pytest.mark.parametrize("base,shape", [("w_qkv", (3 * 64, 64)), ("b_qkv", (3 * 64,)), ("w_fc1", (4 * 64, 64)),
                                        ("b_fc1", (4 * 64,)), ("w_proj", (64, 64)), ("w_fc2", (64, 4 * 64))])
def test_unshard_inverts_the_device_shard_map(tp, base, shape):
    from paper_2406_08756_b200 import executor as ex
    full = np.arange(int(np.prod(shape)), dtype=np.float32).reshape(shape)
    name = "l3." + base
    assert ex.is_tp_sharded(name)
    parts = [_shard(full, base, tp, r) for r in range(tp)]
    assert all(p.size * tp == full.size for p in parts)
    assert np.array_equal(ex.unshard(parts, name), full)


def test_replicated_tensors_are_not_sharded():
    from paper_2406_08756_b200 import executor as ex
    for n in ["wte", "wpe", "w_head", "lnf_g", "l0.ln1_g", "l2.b_proj", "l1.b_fc2", "l0.ln2_b"]:
        assert not ex.is_tp_sharded(n)
        x = np.ones(3)
        assert ex.unshard([x, x], n) is x


def test_oracle_step_with_dropout_differs_from_without():
    """Dropout reaches the loss through the mask, and the same seed reproduces it exactly."""
    from paper_2406_08756_b200 import executor as ex
    from paper_2406_08756_b200 import gpt_profile as gp
    c = gp.GPTConfig("gpt-mini", 1, 64, 2, 16, 2, 256, 1, 1, 1, dropout=0.1)
    shapes = ex.param_shapes(c, 1, True, True)
    rng = np.random.default_rng(0)
    params = {k: (rng.standard_normal(int(np.prod(s))) * 0.02).astype(np.float32) for k, s in shapes.items()}
    for k in params:
        if k.endswith("_g"):
            params[k][:] = 1
    tok, lab = ex.synthetic_batch(c)
    kw = dict(n_layers=1, hidden=64, heads=2, seq=16, micro_batch=2, n_micro=1)
    l0, _ = go.gpt_step(params, shapes, tok, lab, dropout=0.0, **kw)
    l1, g1 = go.gpt_step(params, shapes, tok, lab, dropout=0.1, **kw)
    l2, g2 = go.gpt_step(params, shapes, tok, lab, dropout=0.1, **kw)
    assert l0 != l1 and l1 == l2
    assert all(np.array_equal(g1[k], g2[k]) for k in g1)


def test_vocab_parallel_head_unshards_by_rows():
    from paper_2406_08756_b200 import executor as ex
    from paper_2406_08756_b200 import gpt_profile as gp
    c = gp.GPTConfig("t", 2, 512, 8, 256, 2, 50432, tp=2)
    assert c.vocab_parallel and not gp.GPTConfig("t", 2, 512, 8, 256, 2, 50304, tp=2).vocab_parallel
    assert ex.param_shapes(c, 2, False, True)["w_head"] == (25216, 512)
    full = np.arange(8 * 3, dtype=np.float32).reshape(8, 3)
    assert ex.is_tp_sharded("w_head", True) and not ex.is_tp_sharded("w_head", False)
    assert np.array_equal(ex.unshard([full[:4], full[4:]], "w_head", True), full)
