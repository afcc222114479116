"""Compressed model codec ("FGSC 22-byte model I/O"): compress_model /
decompress_model (io.hpp:319-425), binary16 codec half.hpp:12-52.

Oracle: the UNCHANGED reference io.hpp compiled here (oracle/_ref; its JSON dependency, used
only by the sidecar formats, is a compile-only shim). CPU part: the reference pinned to the
golden bytes of test_io.cpp:170-186, the size formula, idempotence and its header errors,
plus an independent numpy binary16 encoder (round-half-even via float16 where exact).
GPU part: device bytes == reference bytes for random, saturating, subnormal and tiny-
quaternion clouds; decoded clouds bit-identical to the reference's (incl. crafted halves:
zero / negative / subnormal / inf / NaN scales, negative densities, zero quaternions);
header errors with the reference's messages and offsets. Note: compress(decompress(b)) == b
holds for the reference's test cloud but not for every splat -- in 4 of 5000 random splats a
small quaternion component moves by a few binary16 ulps (the quantize-then-renormalise fixed
point is not unique); the device codec reproduces the reference's bytes there too."""
from __future__ import annotations

import numpy as np
import pytest

from oracle.oracle import OracleError
from paper_2604_01844_b200 import gsct


def _params(c: gsct.GaussianCloud) -> dict:
    return {"pos": c.positions, "ls": c.log_scales, "q": c.rotations, "raw": c.raw_densities}


def _clouds():
    out = {}
    for m in (1, 3, 40, 257, 5000):
        out[f"random{m}"] = gsct.make_cloud("random", m, seed=40 + m)
    c = gsct.make_cloud("random", 300, seed=7)
    c.positions[:10] *= 3e4       # |x| >= 65520 saturates
    c.log_scales[10:20] = -20.0   # subnormal-range scales
    c.log_scales[20:25] = 12.0    # scales past 65504
    c.rotations[25:35] *= 1e-6    # tiny (unnormalised) quaternions
    c.rotations[35:40] = [1e-3, 1.0, -1.0, 1e-3]
    c.raw_densities[40:50] = -0.5  # activated density 0
    c.raw_densities[50:55] = 7e4   # saturating density
    out["extremes"] = c
    return out


def test_reference_codec_pinned(ref):
    one = {"pos": np.array([[0.0, 0.5, -2.0]]), "ls": np.zeros((1, 3)), "q": np.array([[1.0, 0, 0, 0]]),
           "raw": np.array([1.0])}
    b, sat = ref.compress_model(one)
    assert bytes(b[:4]) == b"FGSC" and b[4] == 1 and b[8] == 1 and len(b) == 38 and sat == 0
    assert list(b[16:]) == [0x00, 0x00, 0x00, 0x38, 0x00, 0xc0, 0x00, 0x3c, 0x00, 0x3c, 0x00, 0x3c,
                            0x00, 0x3c, 0x00, 0x00, 0x00, 0x00, 0x00, 0x00, 0x00, 0x3c]  # test_io.cpp:176-182
    # idempotent at binary16 precision (test_io.cpp:189-194: random_cloud(44, 25))
    c44 = gsct.make_cloud("random", 25, seed=44)
    b, _ = ref.compress_model(_params(c44))
    assert np.array_equal(b, ref.compress_model(ref.decompress_model(b, 25))[0])
    for name, c in _clouds().items():
        b, sat = ref.compress_model(_params(c))
        assert len(b) == 16 + 22 * c.size()
        # positions and densities: the numpy half encoder (round-half-even) agrees
        h = b[16:].view("<u2").reshape(-1, 11)
        pos16 = np.clip(c.positions, -65504, 65504).astype(np.float16).view("<u2")
        assert np.array_equal(h[:, :3], pos16), name
    with pytest.raises(OracleError, match=r"bad magic.*\(byte offset 0\)"):
        ref.decompress_model(np.frombuffer(b"XGSC" + bytes(12), dtype=np.uint8))


@pytest.mark.gpu
@pytest.mark.parametrize("name", list(_clouds().keys()))
def test_compress_matches_reference(ref, ctx, name):
    c = _clouds()[name]
    want, wsat = ref.compress_model(_params(c))
    got, sat = gsct.compress_model(c, ctx=ctx)  # host buffers
    assert sat == wsat
    assert np.array_equal(got, want)
    dgot, dsat = gsct.compress_model(c.to_device(0), ctx=ctx)  # device-resident
    assert dsat == wsat and np.array_equal(dgot.cpu().numpy(), want)
    # decode: bit-identical to the reference (log-scales from the glibc table)
    r = ref.decompress_model(want, c.size())
    # re-compressing the decoded cloud: the reference's bytes, quirks included
    re_want, _ = ref.compress_model(r)
    re_got, _ = gsct.compress_model(gsct.GaussianCloud(r["pos"], r["ls"], r["q"], r["raw"]), ctx=ctx)
    assert np.array_equal(re_got, re_want)
    for cloud in (gsct.decompress_model(want, ctx=ctx), gsct.decompress_model(dgot, ctx=ctx).numpy()):
        assert np.array_equal(cloud.positions, r["pos"])
        assert np.array_equal(cloud.log_scales, r["ls"])
        assert np.array_equal(cloud.rotations, r["q"])
        assert np.array_equal(cloud.raw_densities, r["raw"])


@pytest.mark.gpu
def test_decompress_crafted_halves(ref, ctx):
    rng = np.random.default_rng(3)
    n = 4096
    words = rng.integers(0, 1 << 16, size=(n, 11), dtype=np.uint64).astype(np.uint16)
    special = np.array([0x0000, 0x8000, 0x0001, 0x03ff, 0x0400, 0x7bff, 0x7c00, 0xfc00, 0x7e00, 0xfe00, 0xbc00],
                       dtype=np.uint16)
    words[: len(special), 3:6] = special[:, None]
    words[: len(special), 10] = special
    words[len(special):len(special) + 8, 6:10] = 0  # zero quaternion -> identity
    data = np.concatenate([np.frombuffer(b"FGSC", dtype=np.uint8), np.array([1, 0, 0, 0], dtype=np.uint8),
                           np.frombuffer(np.uint64(n).tobytes(), dtype=np.uint8), words.view(np.uint8).ravel()])
    r = ref.decompress_model(data, n)
    got = gsct.decompress_model(data, ctx=ctx)
    for a, k in ((got.positions, "pos"), (got.log_scales, "ls"), (got.rotations, "q"), (got.raw_densities, "raw")):
        assert np.array_equal(a, r[k], equal_nan=True), k


@pytest.mark.gpu
def test_decompress_header_errors_match_reference(ref, ctx):
    good, _ = ref.compress_model(_params(gsct.make_cloud("random", 4, seed=46)))
    cases = {
        "truncated body": good[:-3],
        "bad magic": np.concatenate([np.frombuffer(b"X", dtype=np.uint8), good[1:]]),
        "short header": good[:10],
        "no magic": good[:2],
        "version": np.concatenate([good[:4], np.array([2, 0, 0, 0], dtype=np.uint8), good[8:]]),
        "trailing": np.concatenate([good, np.zeros(5, dtype=np.uint8)]),
    }
    for name, data in cases.items():
        with pytest.raises(OracleError) as want:
            ref.decompress_model(data)
        with pytest.raises(gsct.ParseError) as got:
            gsct.decompress_model(data, ctx=ctx)
        assert str(got.value) == str(want.value), name
    assert gsct.decompress_model(good[:16] * 0 + np.frombuffer(b"FGSC" + bytes([1, 0, 0, 0]) + bytes(8), dtype=np.uint8),
                                 ctx=ctx).size() == 0


@pytest.mark.gpu
def test_compress_contract(ctx):
    c = gsct.make_cloud("random", 20, seed=1)
    c.rotations[7] = 0.0
    with pytest.raises(gsct.ContractError, match="zero quaternion in splat 7"):
        gsct.compress_model(c, ctx=ctx)


@pytest.mark.gpu
def test_empty_model_roundtrip(ref, ctx):
    """test_io.cpp:152-161: an empty cloud is exactly the 16-byte header."""
    b, sat = gsct.compress_model(gsct.GaussianCloud.empty(), ctx=ctx)
    want, _ = ref.compress_model({"pos": np.zeros((0, 3)), "ls": np.zeros((0, 3)), "q": np.zeros((0, 4)),
                                  "raw": np.zeros(0)})
    assert sat == 0 and len(b) == 16 and np.array_equal(b, want) and bytes(b[:4]) == b"FGSC"
    assert gsct.decompress_model(b, ctx=ctx).size() == 0
