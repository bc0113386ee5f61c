"""Golden fixtures for the `.pwix` container and CRC-32C, made by
the reference itself.

Run once in the build container (where /root/reference exists):

    python tests/golden/make_golden_container.py

Writes tests/golden/container.npz:
* crc_<n>                 shardann._crc32c.crc32c of pattern_bytes(n) (serial
                          path below 16 KiB, lane path above)
* comb_*                  crc32c_combine cases
* small_pwix              the bytes shardann.serialize_index writes for the
                          conftest small_index (4 shards, d=16, ghost +
                          direction + inter-shard tables), and small_file_crc
                          = index_file_checksum of it
* bare_pwix               the same for a 1-shard index without optional
                          sections (test_container.py:91-101)

Nothing at test time reads /root/reference.
"""

from __future__ import annotations

import sys
import tempfile
from pathlib import Path

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
import shardann as sa  # noqa: E402
from shardann._crc32c import crc32c, crc32c_combine  # noqa: E402

OUT = Path(__file__).resolve().parent
SIZES = (0, 1, 3, 9, 100, 4095, 16383, 16384, 16385, 70_001, 500_000, 1 << 20)


def pattern_bytes(n: int, salt: int = 0) -> np.ndarray:
    """Deterministic pseudo-random bytes (splitmix64 finaliser of the index);
    tests/test_container.py regenerates them instead of storing them."""
    with np.errstate(over="ignore"):
        z = np.arange(n, dtype=np.uint64) + np.uint64(salt) * np.uint64(0x9E3779B97F4A7C15)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        z = z ^ (z >> np.uint64(31))
    return (z >> np.uint64(24)).astype(np.uint8)


def main():
    out = {}
    for n in SIZES:
        out[f"crc_{n}"] = np.uint32(crc32c(pattern_bytes(n)))
    comb = []
    for n1, n2 in ((0, 5), (5, 0), (777, 9223), (1 << 16, 12345), (3, 1 << 20)):
        a = pattern_bytes(n1, 1).tobytes()
        b = pattern_bytes(n2, 2).tobytes()
        comb.append((crc32c(a), crc32c(b), n2, crc32c_combine(crc32c(a), crc32c(b), n2)))
    out["comb"] = np.array(comb, dtype=np.uint64)

    full = sa.gen_synthetic(4100, 16, 32, 0.2, seed=99)  # conftest.py small_data
    base = sa.Dataset(full.data[:4000])
    small, _ = sa.build_index(base, 4, 16, seed=5, rho=0.05, ghost_degree=8)  # small_index
    bare, _ = sa.build_index(base, 1, 8, seed=1, with_ghost=False, with_direction=False)
    with tempfile.TemporaryDirectory() as td:
        for name, index in (("small", small), ("bare", bare)):
            path = Path(td) / f"{name}.pwix"
            sa.serialize_index(index, path)
            out[f"{name}_pwix"] = np.frombuffer(path.read_bytes(), np.uint8)
            out[f"{name}_file_crc"] = np.array(sa.index_file_checksum(path))
    np.savez_compressed(OUT / "container.npz", **out)
    print({k: v.shape for k, v in out.items()})


if __name__ == "__main__":
    main()
