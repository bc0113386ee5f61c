"""`.pwix` container + CRC-32C, mirroring the reference's
tests/test_container.py (KATs :13-16, lane path :19-23, combine :26-31, round
trip :34-39, corruption :42-51, version :54-62, magic :65-69, truncation
:72-79, optional sections :82-92, file checksum :95-101), pinned to bytes and
CRCs the reference itself produced (tests/golden/make_golden_container.py).

CPU tests: oracle and host CRC against the goldens, serializer byte-identity,
error behaviour.  GPU tests: the CRC kernel (K3) against the oracle at
aligned/unaligned offsets and sizes up to 1 GiB, and the device load path.
"""

from __future__ import annotations

from pathlib import Path

import numpy as np
import pytest

import oracle
import paper_2507_17094_b200 as pw
from paper_2507_17094_b200.container import FORMAT_VERSION, ChecksumError, IndexFormatError, VersionError
import golden_util as gu

GOLDEN = Path(__file__).resolve().parent / "golden"


def _pattern_bytes():
    # the generator's byte pattern without importing the reference
    src = (GOLDEN / "make_golden_container.py").read_text()
    ns: dict = {"np": np}
    start = src.index("def pattern_bytes")
    end = src.index("\n\n\ndef main")
    exec(src[start:end], ns)  # noqa: S102 -- committed fixture code
    return ns["pattern_bytes"]


pattern_bytes = _pattern_bytes()
Z = np.load(GOLDEN / "container.npz")
SIZES = sorted(int(k[4:]) for k in Z.files if k.startswith("crc_"))


@pytest.fixture(scope="module")
def small_index():
    return gu.load("small")[3]


# ------------------------------------------------------------------ CPU tests


def test_oracle_crc_matches_reference_goldens():
    assert oracle.crc32c(b"123456789") == 0xE3069283
    assert oracle.crc32c(b"") == 0
    assert oracle.crc32c(b"\x00" * 32) == 0x8A9136AA
    for n in SIZES:
        assert oracle.crc32c(pattern_bytes(n)) == int(Z[f"crc_{n}"]), n


def test_crc32c_known_answer():
    assert pw.crc32c(b"123456789") == 0xE3069283
    assert pw.crc32c(b"") == 0
    assert pw.crc32c(b"\x00" * 32) == 0x8A9136AA


def test_host_crc_matches_reference_goldens():
    for n in SIZES:
        assert pw.crc32c(pattern_bytes(n)) == int(Z[f"crc_{n}"]), n


def test_host_crc_threads_and_offsets_match_oracle():
    buf = pattern_bytes((40 << 20) + 13, 7)  # above the 8 MB/thread split
    want = oracle.crc32c(buf)
    for threads in (1, 2, 5, 0):
        assert pw.crc32c(buf, threads=threads) == want, threads
    for off in (1, 3, 7):  # unaligned starts
        assert pw.crc32c(buf[off:off + 100_003]) == oracle.crc32c(buf[off:off + 100_003])


def test_crc32c_combine_matches_reference():
    for c1, c2, n2, want in Z["comb"]:
        assert pw.crc32c_combine(int(c1), int(c2), int(n2)) == int(want)
    whole = pattern_bytes(10_000, 3).tobytes()
    for cut in (0, 1, 777, 9_999, 10_000):
        a, b = whole[:cut], whole[cut:]
        assert pw.crc32c_combine(pw.crc32c(a), pw.crc32c(b), len(b)) == pw.crc32c(whole)


def test_serialize_is_byte_identical_to_reference(tmp_path, small_index):
    path = tmp_path / "idx.pwix"
    pw.serialize_index(small_index, path)
    assert path.read_bytes() == Z["small_pwix"].tobytes()
    assert pw.index_file_checksum(path) == str(Z["small_file_crc"])


def test_deserialize_reference_file(tmp_path, small_index):
    path = tmp_path / "ref.pwix"
    path.write_bytes(Z["small_pwix"].tobytes())
    loaded = pw.deserialize_index(path)
    assert pw.index_equal(small_index, loaded)
    assert loaded.shards[0].direction.dtype == np.uint32 and loaded.shards[0].adj.dtype == np.int32


def test_bare_index_round_trip(tmp_path):
    path = tmp_path / "bare.pwix"
    path.write_bytes(Z["bare_pwix"].tobytes())
    loaded = pw.deserialize_index(path)
    pack = loaded.shards[0]
    assert pack.inter_map is None and pack.ghost_ids is None and pack.direction is None
    out = tmp_path / "bare2.pwix"
    pw.serialize_index(loaded, out)
    assert out.read_bytes() == Z["bare_pwix"].tobytes()
    assert pw.index_file_checksum(out) == str(Z["bare_file_crc"])


def test_corrupted_byte_fails_checksum(tmp_path):
    blob = bytearray(Z["small_pwix"].tobytes())
    blob[-1] ^= 0xFF
    path = tmp_path / "bad.pwix"
    path.write_bytes(bytes(blob))
    with pytest.raises(ChecksumError, match="checksum mismatch"):
        pw.deserialize_index(path)


def test_future_version_rejected(tmp_path):
    blob = bytearray(Z["small_pwix"].tobytes())
    blob[4:8] = (FORMAT_VERSION + 1).to_bytes(4, "little")
    path = tmp_path / "v.pwix"
    path.write_bytes(bytes(blob))
    with pytest.raises(VersionError, match="version"):
        pw.deserialize_index(path)


def test_bad_magic_rejected(tmp_path):
    path = tmp_path / "junk.pwix"
    path.write_bytes(b"NOPE" + b"\x00" * 60)
    with pytest.raises(IndexFormatError, match="magic"):
        pw.deserialize_index(path)


def test_truncated_container_rejected(tmp_path):
    blob = Z["small_pwix"].tobytes()
    for cut in (10, 30, len(blob) // 2, len(blob) - 1):
        path = tmp_path / f"t{cut}.pwix"
        path.write_bytes(blob[:cut])
        with pytest.raises(IndexFormatError):
            pw.deserialize_index(path)


def test_errors_are_value_errors():
    assert issubclass(ChecksumError, IndexFormatError) and issubclass(VersionError, IndexFormatError)
    assert issubclass(IndexFormatError, ValueError)


# ------------------------------------------------------------------ GPU tests


@pytest.mark.gpu
def test_device_crc_matches_oracle_and_goldens():
    import torch

    dev = torch.device("cuda")
    for n in SIZES:
        t = torch.from_numpy(pattern_bytes(n)).to(dev)
        assert pw.crc32c_device([t]) == [int(Z[f"crc_{n}"])], n
    # many sections of one launch, unaligned starts and ragged lengths
    buf = pattern_bytes((3 << 20) + 77, 11)
    dbuf = torch.from_numpy(buf).to(dev)
    cuts = [(0, 0), (1, 1), (3, 15), (5, 16), (16, 17), (4, 8191), (13, 8192 + 33), (100, 300_001),
            (7, (3 << 20) + 70), (0, (3 << 20) + 77)]
    got = pw.crc32c_device([dbuf[a:a + n] for a, n in cuts])
    assert got == [oracle.crc32c(buf[a:a + n]) for a, n in cuts]


@pytest.mark.gpu
def test_device_crc_large_buffer_matches_host():
    import torch

    n = (1 << 30) + 12_345  # 1 GiB: many tiles per lane, constant-gap folding
    t = torch.randint(0, 256, (n,), dtype=torch.uint8, device="cuda")
    host = t.cpu().numpy()
    assert pw.crc32c_device([t]) == [pw.crc32c(host)]
    assert pw.crc32c_device([t[3:]]) == [pw.crc32c(host[3:])]


@pytest.mark.gpu
def test_load_index_device_reference_file(tmp_path, small_index):
    import torch

    path = tmp_path / "ref.pwix"
    path.write_bytes(Z["small_pwix"].tobytes())
    di = pw.load_index_device(path)
    assert (di.d, di.n_total, di.n_shards) == (small_index.d, small_index.n_total, small_index.n_shards)
    for sh, pack in zip(di.shards, small_index.shards):
        for name in ("global_ids", "adj", "inter_map", "ghost_ids", "ghost_adj", "direction"):
            want = getattr(pack, name)
            got = sh.get(name)
            assert (got is None) == (want is None), name
            if want is not None:
                assert np.array_equal(got.cpu().numpy().view(want.dtype), want), name
    blob = bytearray(Z["small_pwix"].tobytes())
    blob[-1] ^= 0x01
    bad = tmp_path / "bad.pwix"
    bad.write_bytes(bytes(blob))
    with pytest.raises(ChecksumError, match="checksum mismatch"):
        pw.load_index_device(bad)
    torch.cuda.synchronize()


@pytest.mark.gpu
def test_device_loaded_index_searches_like_reference(tmp_path):
    """Shards built from the device-loaded container reproduce the reference's
    pipelined run on the golden fixture (ids, distances, counters)."""
    import torch

    from paper_2507_17094_b200 import device as D

    z, base, queries, index, _ = gu.load("small")
    path = tmp_path / "ref.pwix"
    path.write_bytes(Z["small_pwix"].tobytes())
    di = pw.load_index_device(path)
    vec = torch.from_numpy(np.ascontiguousarray(base.data)).cuda()
    shards = di.tensor_shards(vec)
    name, params, mode, prefix = next(c for c in gu.small_cases() if c[2] == "pipelined")
    q = torch.from_numpy(queries).cuda()
    run = D.DeviceRun(q.shape[0], len(shards), params.k, q.device)
    D.run_local(shards, params, q, mode, run)
    torch.cuda.synchronize()
    want = gu.expected(z, prefix)
    assert np.array_equal(run.final_ids.cpu().numpy(), want["final_ids"])
    assert np.array_equal(run.final_dists.cpu().numpy(), want["final_dists"])
