"""CPU: host-side logic of the drop-in API (validation, constants, flush
schedule, byte accounting) — everything that runs before a kernel launch."""
import numpy as np
import pytest

import paper_2510_05373_b200 as qk
from oracle import kvlinc_oracle as orc
from paper_2510_05373_b200.batched import flush_count


def test_config_validation_messages():
    with pytest.raises(ValueError, match="bits"):
        qk.QuantConfig(bits=5)
    with pytest.raises(ValueError, match="group_size"):
        qk.QuantConfig(group_size=0)
    with pytest.raises(ValueError, match="axis"):
        qk.QuantConfig(axis="row")
    with pytest.raises(ValueError, match="rotation"):
        qk.QuantConfig(rotation="both")
    assert qk.QuantConfig(bits=16).is_passthrough
    assert qk.QuantConfig(axis="channel", rotation="post").label() == "channel/post"


def test_pack_and_group_validation_before_device():
    with pytest.raises(ValueError, match="range"):
        qk.pack_codes(np.array([4]), bits=2)
    with pytest.raises(ValueError, match="range"):
        qk.pack_codes(np.array([-1]), bits=2)
    with pytest.raises(ValueError, match="pack"):
        qk.pack_codes(np.array([0]), bits=16)
    with pytest.raises(ValueError, match="exceeds capacity"):
        qk.unpack_codes(np.array([0], dtype=np.uint32), 17, bits=2)
    with pytest.raises(ValueError, match="non-empty"):
        qk.quantize_group([], bits=2)
    with pytest.raises(ValueError, match="bits"):
        qk.quantize_group([1.0, 2.0], bits=16)
    with pytest.raises(ValueError, match="scale"):
        qk.dequantize_group(np.array([0]), -1.0, 0.0)
    with pytest.raises(ValueError, match="passthrough"):
        qk.quantize_tensor(np.ones((2, 2)), qk.QuantConfig(bits=16))
    with pytest.raises(ValueError, match="non-empty"):
        qk.quantize_tensor(np.ones((0, 2)), qk.QuantConfig())
    assert qk.expected_quant_mse(1.0) == pytest.approx(1.0 / 12.0)


def test_hadamard_matrix_is_the_reference_constant(golden):
    for dim in (2, 4, 8, 16, 32, 64, 128, 256):
        assert np.array_equal(qk.hadamard_matrix(dim).matrix, golden["hadamard"][f"H/{dim}"])
    for dim in (0, 3, 12, 100):
        with pytest.raises(ValueError, match="power of two"):
            qk.hadamard_matrix(dim)
    with pytest.raises(ValueError, match="placement"):
        qk.rotate(np.zeros((4, 4)), qk.hadamard_matrix(4), "sideways")
    with pytest.raises(ValueError, match="rows"):
        qk.rotate(np.zeros((8, 4)), qk.hadamard_matrix(4), "pre")


def test_adapter_initialisation_matches_reference(golden):
    z = golden["adapter"]
    ad = qk.CorrectionAdapter.initialize(128, 256, seed=5)
    for n in ("w1_q", "w2_q", "w1_k", "w2_k"):
        assert np.array_equal(getattr(ad, n), z[f"ad/128_256_5/{n}"])
    assert ad.rank == 256 and ad.head_dim == 128
    with pytest.raises(ValueError, match="rank"):
        qk.CorrectionAdapter.initialize(8, 3)
    with pytest.raises(ValueError, match="shapes"):
        qk.CorrectionAdapter(np.zeros((2, 2)), np.zeros((2, 2)), np.zeros((2, 2)), np.zeros((3, 2)))


def test_cache_constructor_validation_and_empty_footprint():
    with pytest.raises(ValueError, match="head_dim"):
        qk.KVCacheState(0)
    with pytest.raises(ValueError, match="group_size"):
        qk.KVCacheState(8, group_size=0)
    with pytest.raises(ValueError, match="residual_window"):
        qk.KVCacheState(8, residual_window=-1)
    with pytest.raises(ValueError, match="power of two"):
        qk.KVCacheState(12, rotate_values=True)
    c = qk.KVCacheState(12, rotate_values=False)
    assert c.quantized_tokens == 0 and c.residual_len == 0 and c.value_rows is None
    assert qk.memory_footprint(qk.KVCacheState(8)).total == 0


@pytest.mark.parametrize("n", [0, 1, 127, 128, 255, 256, 383, 384, 1000, 8192, 131072])
def test_flush_schedule_equals_streaming_rule(n):
    """Host mirror of the flush rule == the reference's append/flush loop (cache.py:120-130)."""
    res, flushed = 0, 0
    for _ in range(min(n, 5000)):
        res += 1
        if res == 128 + 128:
            res -= 128
            flushed += 1
    if n <= 5000:
        assert flush_count([n])[0] == flushed
        assert n - 128 * flush_count([n])[0] == res
    assert flush_count([n], keep_window=False)[0] == n // 128


def test_byte_accounting_matches_reference_closed_form(golden):
    """memory_footprint tally of the reference (c11: 646,144 B at 8192 tokens, d=G=R=128)."""
    z = golden["cache"]
    for name in ("c_small", "c_rot", "c_prod"):
        n, d, g, win, rot, rank = (int(x) for x in z[f"{name}/meta"][:6])
        nq, nr = int(z[f"{name}/meta"][7]), int(z[f"{name}/meta"][8])
        lanes = 16
        chunks = nq // g
        codes = 4 * (chunks * -(-g // lanes) * d + nq * -(-d // lanes))
        meta = 2 * 2 * (chunks * d + nq * -(-d // g))
        states = 2 * (d * rank + rank) if rank else 0
        assert [codes, meta, 2 * 2 * nr * d, states] == list(z[f"{name}/footprint"])
    nq = 8192 - 128
    assert 4 * (nq // 128 * 8 * 128 + nq * 8) + 4 * (nq // 128 * 128 + nq) + 4 * 128 * 128 == 646144


def test_oracle_gqa_wrapper_shapes():
    g = orc.rng(0)
    caches = [[orc.build_cache(g.standard_normal((300, 16)), g.standard_normal((300, 16)),
                               group=32, window=32)]]
    out = orc.decode_gqa(g.standard_normal((1, 2, 16)), caches, None)
    assert out.shape == (1, 2, 16) and np.all(np.isfinite(out))


def test_kvlc_format_round_trips_reference_bytes(golden):
    """Host side of the .kvlc format (paper_2510_05373_b200/kvlc_format.py): the
    parsed sections re-join to the reference's bytes; the reader's errors carry
    the reference's messages (cache.py:233-304)."""
    import pytest
    from paper_2510_05373_b200 import kvlc_format as fmt
    z = golden["cache"]
    names = sorted({k.split("/")[0] for k in z if k.endswith("/kvlc")})
    assert "c_prod" in names
    for name in names:
        ref = z[f"{name}/kvlc"].tobytes()
        h = fmt.parse_header(ref)
        assert h.nbytes() == len(ref)
        assert fmt.join(h, fmt.split(ref, h)) == ref, name
    ref = z["c_prod/kvlc"].tobytes()
    with pytest.raises(fmt.CacheFormatError, match="bad magic at byte 0"):
        fmt.parse_header(b"XXXX" + ref[4:])
    with pytest.raises(fmt.CacheFormatError, match="unsupported cache version 2 at byte 4"):
        fmt.parse_header(ref[:4] + (2).to_bytes(4, "little") + ref[8:])
    h = fmt.parse_header(ref)
    with pytest.raises(fmt.CacheFormatError, match="truncated cache file at byte"):
        fmt.split(ref[:-1], h)
    with pytest.raises(fmt.CacheFormatError, match="trailing bytes at byte"):
        fmt.split(ref + b"\0", h)
    assert issubclass(fmt.CacheFormatError, ValueError)


def test_adapter_file_format_matches_reference(golden, tmp_path):
    """.kvla bytes (adapter.py:310-362): host-side format, byte-identical to the reference."""
    import pytest
    from paper_2510_05373_b200 import CorrectionAdapter, train
    want = golden["train"]["t/kvla"].tobytes()
    ad = CorrectionAdapter.initialize(16, 8, seed=4)
    assert train.serialize_adapter(ad) == want
    back = train.deserialize_adapter(want)
    assert train.serialize_adapter(back) == want and back.enabled
    path = tmp_path / "a.kvla"
    train.write_adapter(ad, path)
    assert train.read_adapter(path).rank == 8
    with pytest.raises(train.AdapterFormatError, match="bad magic"):
        train.deserialize_adapter(b"XXXX" + want[4:])
    with pytest.raises(train.AdapterFormatError, match="payload size mismatch"):
        train.deserialize_adapter(want[:-4])
    with pytest.raises(train.AdapterFormatError, match="too short"):
        train.deserialize_adapter(want[:8])
