"""`.pwix` index container (drop-in for shardann/container.py + _crc32c.py).

Same little-endian layout, byte for byte (container.py:1-28): a 24-byte
header, a 28-byte section table entry per section, then the payloads, each
with its CRC-32C.  `serialize_index` output is byte-identical to the
reference's for value-identical indexes (tests/test_container.py checks this
against files the reference wrote).

Two load paths:

* ``deserialize_index(path) -> Index``: host arrays, as the reference returns
  them; section checksums verified by ``pw_crc32c`` (native: SSE4.2 crc32
  instruction, split over host threads).
* ``load_index_device(path, device) -> DeviceIndex``: the B200 path.  The
  whole file goes to HBM in one pinned host->device copy and every section is
  verified there by ONE launch of the CRC kernel (K3, ``pw_crc32c_device``);
  the shards are then built device-to-device (``DeviceIndex.tensor_shards``)
  without the index ever being re-read on the host.

Errors mirror the reference (container.py:48-58): ``IndexFormatError``
(ValueError), ``VersionError``, ``ChecksumError``, with the same messages.
"""

from __future__ import annotations

import ctypes as C
import struct
from dataclasses import dataclass
from pathlib import Path

import numpy as np

from . import _abi
from .graphs import Index, ShardPack

MAGIC = b"PWIX"
FORMAT_VERSION = 1

_K_META, _K_IDS, _K_ADJ, _K_INTER, _K_GHOST_IDS, _K_GHOST_ADJ, _K_DIR = range(1, 8)
_HEADER = struct.Struct("<4sIIIII")
_SECTION = struct.Struct("<IIQQI")


class IndexFormatError(ValueError):
    """Malformed index container (container.py:48-49)."""


class VersionError(IndexFormatError):
    """Container written by an unknown (newer) format version (container.py:52-53)."""


class ChecksumError(IndexFormatError):
    """Section payload does not match its recorded CRC-32C (container.py:56-57)."""


# ------------------------------------------------------------------ CRC-32C --

def _as_bytes(data) -> np.ndarray:
    if isinstance(data, np.ndarray):
        return np.ascontiguousarray(data).view(np.uint8).ravel()
    return np.frombuffer(data, dtype=np.uint8)


def crc32c(data, threads: int = 0) -> int:
    """_crc32c.py:98-130: CRC-32C of bytes or a numpy array's raw memory."""
    buf = _as_bytes(data)
    lib = _abi.load(require_device=False)
    out = C.c_uint32()
    ptr = buf.ctypes.data if buf.size else None
    _abi.check(lib.pw_crc32c(ptr, buf.size, threads, C.byref(out)))
    return int(out.value)


def crc32c_combine(crc1: int, crc2: int, len2: int) -> int:
    """_crc32c.py:85-89: CRC of the concatenation from the CRCs of both parts."""
    lib = _abi.load(require_device=False)
    out = C.c_uint32()
    _abi.check(lib.pw_crc32c_combine(crc1 & 0xFFFFFFFF, crc2 & 0xFFFFFFFF, len2, C.byref(out)))
    return int(out.value)


def crc32c_device(buffers, stream=None) -> list[int]:
    """CRC-32C of device buffers (torch tensors, any dtype, contiguous) with one
    kernel launch; the B200 form of the per-section checks of container.py:117-124."""
    import torch

    lib = _abi.load()
    n = len(buffers)
    if n == 0:
        return []
    ptrs = (C.c_void_p * n)()
    lens = (C.c_int64 * n)()
    for i, b in enumerate(buffers):
        if not b.is_cuda or not b.is_contiguous():
            raise ValueError("crc32c_device needs contiguous CUDA tensors")
        ptrs[i] = b.data_ptr() if b.numel() else None
        lens[i] = b.numel() * b.element_size()
    devs = {b.device for b in buffers}
    if len(devs) != 1:
        raise ValueError("crc32c_device: all buffers must be on one device")
    out = (C.c_uint32 * n)()
    with torch.cuda.device(devs.pop()):
        st = stream if stream is not None else torch.cuda.current_stream()
        _abi.check(lib.pw_crc32c_device(ptrs, lens, n, out, C.c_void_p(st.cuda_stream)))
    return [int(x) for x in out]


# ---------------------------------------------------------------- serialize --

def _has_padded_rows(adj) -> bool:
    """The container's "padded" meta flag (container.py:60-65): some row
    lists a neighbour twice (degree-deficit padding repeats ids).  A row
    repeats an id iff it has fewer distinct values than slots."""
    if adj is None or adj.size == 0:
        return False
    a = np.asarray(adj)
    srt = np.sort(a, axis=1)
    distinct = 1 + np.count_nonzero(np.diff(srt, axis=1), axis=1)
    return bool((distinct < a.shape[1]).any())


def _host(a):
    if a is None:
        return None
    if hasattr(a, "detach"):  # torch tensor (e.g. a GPU-built index)
        a = a.detach().cpu().numpy()
    return np.asarray(a)


def _shard_sections(pack) -> list[tuple[int, np.ndarray]]:
    """container.py:68-93: (kind, little-endian payload) per section."""
    gid, adj = _host(pack.global_ids), _host(pack.adj)
    inter, gids, gadj, dirn = (_host(pack.inter_map), _host(pack.ghost_ids), _host(pack.ghost_adj),
                               _host(pack.direction))
    n_local, j = adj.shape
    g, j_g = gadj.shape if gadj is not None else (0, 0)
    w = dirn.shape[2] if dirn is not None else 0
    padded = _has_padded_rows(adj) or _has_padded_rows(gadj)
    meta = np.array([n_local, j, g, j_g, w, int(inter is not None), int(gids is not None),
                     int(dirn is not None), int(padded)], dtype="<u4")
    sections = [(_K_META, meta), (_K_IDS, gid.astype("<i4")), (_K_ADJ, adj.astype("<i4"))]
    if inter is not None:
        sections.append((_K_INTER, inter.astype("<i4")))
    if gids is not None:
        sections.append((_K_GHOST_IDS, gids.astype("<i4")))
        sections.append((_K_GHOST_ADJ, gadj.astype("<i4")))
    if dirn is not None:
        sections.append((_K_DIR, dirn.astype("<u4")))
    return [(k, np.ascontiguousarray(a)) for k, a in sections]


def serialize_index(index, path) -> None:
    """container.py:96-114: write the index; byte-identical output for
    value-identical indexes."""
    per_shard = [_shard_sections(pack) for pack in index.shards]
    count = sum(len(s) for s in per_shard)
    offset = _HEADER.size + count * _SECTION.size
    table, payloads = [], []
    for shard, sections in enumerate(per_shard):
        for kind, arr in sections:
            table.append((shard, kind, offset, arr.nbytes, crc32c(arr)))
            payloads.append(arr)
            offset += arr.nbytes
    with open(path, "wb") as f:
        f.write(_HEADER.pack(MAGIC, FORMAT_VERSION, index.d, index.n_shards, index.n_total, count))
        for entry in table:
            f.write(_SECTION.pack(*entry))
        for arr in payloads:
            f.write(memoryview(arr.view(np.uint8).ravel()))


# -------------------------------------------------------------- deserialize --

@dataclass(frozen=True)
class _Layout:
    d: int
    n_shards: int
    n_total: int
    by_shard: dict  # shard -> kind -> (shard, kind, offset, length, crc)


def _parse(blob, path) -> _Layout:
    """container.py:127-150: header + section table checks (host bytes)."""
    if len(blob) < _HEADER.size:
        raise IndexFormatError(f"{path}: too short for a header")
    magic, version, d, n_shards, n_total, count = _HEADER.unpack_from(blob, 0)
    if magic != MAGIC:
        raise IndexFormatError(f"{path}: bad magic {bytes(magic)!r}, not an index container")
    if version > FORMAT_VERSION:
        raise VersionError(f"{path}: format version {version} is newer than supported {FORMAT_VERSION}")
    table_end = _HEADER.size + count * _SECTION.size
    if len(blob) < table_end:
        raise IndexFormatError(f"{path}: truncated section table")
    by_shard: dict[int, dict[int, tuple]] = {}
    for i in range(count):
        entry = _SECTION.unpack_from(blob, _HEADER.size + i * _SECTION.size)
        by_shard.setdefault(entry[0], {})[entry[1]] = entry
    return _Layout(int(d), int(n_shards), int(n_total), by_shard)


def _check_extent(entry, size, path) -> None:
    shard, kind, offset, length, _ = entry
    if offset + length > size:
        raise IndexFormatError(f"{path}: truncated section (shard {shard}, kind {kind})")


def _shard_sections_of(lay: _Layout, s: int, path) -> dict:
    sections = lay.by_shard.get(s)
    if sections is None or _K_META not in sections:
        raise IndexFormatError(f"{path}: missing sections for shard {s}")
    return sections


def _meta(blob, entry, path) -> tuple:
    _check_extent(entry, len(blob), path)
    _, _, offset, length, crc = entry
    raw = np.frombuffer(blob, np.uint8, length, offset)
    if crc32c(raw) != crc:
        raise ChecksumError(f"{path}: checksum mismatch in section (shard {entry[0]}, kind {entry[1]})")
    return tuple(int(x) for x in raw.view("<u4")[:8])


def _shard_plan(sections, meta):
    """(name, kind, dtype, shape) of every array section a shard carries."""
    n_local, j, g, j_g, w, has_inter, has_ghost, has_dir = meta
    plan = [("global_ids", _K_IDS, "<i4", (n_local,)), ("adj", _K_ADJ, "<i4", (n_local, j))]
    if has_inter:
        plan.append(("inter_map", _K_INTER, "<i4", (n_local,)))
    if has_ghost:
        plan.append(("ghost_ids", _K_GHOST_IDS, "<i4", (g,)))
        plan.append(("ghost_adj", _K_GHOST_ADJ, "<i4", (g, j_g)))
    if has_dir:
        plan.append(("direction", _K_DIR, "<u4", (n_local, j, w)))
    return plan


def deserialize_index(path) -> Index:
    """container.py:127-166: read and verify a container; inverse of
    serialize_index."""
    blob = Path(path).read_bytes()
    lay = _parse(blob, path)
    packs = []
    for s in range(lay.n_shards):
        sections = _shard_sections_of(lay, s, path)
        meta = _meta(blob, sections[_K_META], path)
        arrays = {}
        for name, kind, dt, shape in _shard_plan(sections, meta):
            entry = sections[kind]
            _check_extent(entry, len(blob), path)
            _, _, offset, length, crc = entry
            raw = np.frombuffer(blob, np.uint8, length, offset)
            if crc32c(raw) != crc:
                raise ChecksumError(f"{path}: checksum mismatch in section (shard {s}, kind {kind})")
            arrays[name] = raw.view(dt).copy().reshape(shape)
        packs.append(ShardPack(arrays["global_ids"], arrays["adj"], arrays.get("inter_map"),
                               arrays.get("ghost_ids"), arrays.get("ghost_adj"), arrays.get("direction")))
    return Index(d=lay.d, n_total=lay.n_total, shards=packs)


@dataclass
class DeviceIndex:
    """A verified container resident in HBM: per shard a dict of int32/uint32
    device tensors (views into the one uploaded blob), shaped as ShardPack."""

    d: int
    n_total: int
    shards: list
    blob: object  # the device copy of the file (the views keep it alive)

    @property
    def n_shards(self) -> int:
        return len(self.shards)

    def tensor_shards(self, vectors) -> list:
        """TensorShards for search (device.TensorShard); ``vectors`` is the
        (n_total, d) device dataset indexed by global id.  Rows are gathered
        on the device (pipeline.py:138-148)."""
        from .device import TensorShard

        out = []
        for sh in self.shards:
            rows = vectors.index_select(0, sh["global_ids"].long())
            out.append(TensorShard(rows, sh["adj"], sh["global_ids"], sh.get("direction"),
                                   sh.get("inter_map"), sh.get("ghost_ids"), sh.get("ghost_adj")))
        return out


def load_index_device(path, device=None) -> DeviceIndex:
    """Read a container straight into HBM and verify every section there with
    one CRC kernel launch (K3).  Same checks and errors as deserialize_index."""
    import torch

    _abi.load()
    dev = torch.device("cuda", torch.cuda.current_device() if device is None else device)
    path = Path(path)
    size = path.stat().st_size
    host = torch.empty(size, dtype=torch.uint8, pin_memory=True)
    with open(path, "rb") as f:
        f.readinto(memoryview(host.numpy()))
    blob = host.numpy()
    lay = _parse(blob, path)
    with torch.cuda.device(dev):
        stream = torch.cuda.current_stream()
        dblob = torch.empty(size, dtype=torch.uint8, device=dev)
        dblob.copy_(host, non_blocking=True)
        metas, plans, checks = [], [], []
        for s in range(lay.n_shards):
            sections = _shard_sections_of(lay, s, path)
            meta = _meta(blob, sections[_K_META], path)  # 36 bytes: checked on the host
            plan = _shard_plan(sections, meta)
            for name, kind, dt, shape in plan:
                entry = sections[kind]
                _check_extent(entry, size, path)
                expect = int(np.prod(shape)) * 4
                if entry[3] != expect:
                    raise IndexFormatError(f"{path}: section (shard {s}, kind {kind}) has {entry[3]} bytes,"
                                           f" expected {expect}")
                checks.append((s, kind, entry))
            metas.append(meta)
            plans.append(plan)
        got = crc32c_device([dblob[e[2]:e[2] + e[3]] for _, _, e in checks], stream)
        for (s, kind, e), c in zip(checks, got):
            if c != e[4]:
                raise ChecksumError(f"{path}: checksum mismatch in section (shard {s}, kind {kind})")
        shards = []
        for s in range(lay.n_shards):
            sh = {}
            for name, kind, dt, shape in plans[s]:
                e = lay.by_shard[s][kind]
                sh[name] = dblob[e[2]:e[2] + e[3]].view(torch.int32).view(shape)
            shards.append(sh)
    return DeviceIndex(d=lay.d, n_total=lay.n_total, shards=shards, blob=dblob)


def index_equal(a, b) -> bool:
    """container.py:169-182: value equality over every array of two indexes."""
    def arr_eq(x, y):
        if x is None or y is None:
            return x is None and y is None
        x, y = _host(x), _host(y)
        return x.shape == y.shape and bool(np.array_equal(x, y))

    if (a.d, a.n_total, a.n_shards) != (b.d, b.n_total, b.n_shards):
        return False
    for pa, pb in zip(a.shards, b.shards):
        for name in ("global_ids", "adj", "inter_map", "ghost_ids", "ghost_adj", "direction"):
            if not arr_eq(getattr(pa, name), getattr(pb, name)):
                return False
    return True


def index_file_checksum(path) -> str:
    """container.py:185-188 (index_file_checksum): CRC-32C of the whole file, hex."""
    return f"{crc32c(np.fromfile(path, dtype=np.uint8)):08x}"
