"""TCRVTEN / TCRVMSK file formats (reference: tokencarve tensorio.py), device-aware.

Header (both formats): 8-byte magic, uint8 version (1), uint8 rank, rank x little-endian
uint64 axis lengths.  Tensor body: row-major little-endian float32.  Mask body: each
last-axis row bit-packed big-endian (np.packbits order), padded to a byte.  Files are
byte-identical to the reference's (round trips are bit-exact both ways).

Device side: ``write_mask`` of a :class:`BlockMask` packs the rows on the GPU straight
from its uint32 words (``tcb_mask_words_to_packbits``), and ``read_block_mask`` unpacks
a file on the GPU into the packed words + row counts the attention kernels read, so a mask file
never exists as a dense bool array on the host.  Tensors may be numpy arrays or torch
tensors (CUDA tensors are copied to the host once).
"""

from __future__ import annotations

import struct
from pathlib import Path

import numpy as np
import torch

from . import _dev, _native
from .errors import ParseError, ShapeError

__all__ = ["write_tensor", "read_tensor", "write_mask", "read_mask", "read_block_mask",
           "TENSOR_MAGIC", "MASK_MAGIC"]

TENSOR_MAGIC = b"TCRVTEN\x00"
MASK_MAGIC = b"TCRVMSK\x00"
VERSION = 1
MAX_RANK = 8


def _header(magic: bytes, shape) -> bytes:
    if len(shape) > MAX_RANK:
        raise ShapeError(f"rank {len(shape)} exceeds the format limit {MAX_RANK}")
    return magic + struct.pack("<BB", VERSION, len(shape)) + struct.pack(f"<{len(shape)}Q", *shape)


def _parse_header(buf: bytes, magic: bytes, path):
    if buf[:8] != magic:
        raise ParseError(f"bad magic {bytes(buf[:8])!r}, expected {magic!r}", path, 0)
    if len(buf) < 10:
        raise ParseError("truncated header", path, 8)
    version, rank = struct.unpack_from("<BB", buf, 8)
    if version != VERSION:
        raise ParseError(f"unsupported version {version}", path, 8)
    if rank > MAX_RANK:
        raise ParseError(f"rank {rank} exceeds the format limit {MAX_RANK}", path, 9)
    end = 10 + 8 * rank
    if len(buf) < end:
        raise ParseError("truncated axis lengths", path, 10)
    return struct.unpack_from(f"<{rank}Q", buf, 10), end


def _host(arr) -> np.ndarray:
    if isinstance(arr, torch.Tensor):
        return arr.detach().cpu().numpy()
    return np.asarray(arr)


def write_tensor(path, arr) -> None:
    """float32 tensor file; other real dtypes are cast to float32 (tensorio.py:60-65)."""
    a = np.ascontiguousarray(_host(arr).astype("<f4", copy=False))
    with open(path, "wb") as fh:
        fh.write(_header(TENSOR_MAGIC, a.shape))
        fh.write(a.tobytes())


def read_tensor(path, device=None):
    """numpy float32 array (or a tensor on ``device``) (tensorio.py:68-77)."""
    path = Path(path)
    buf = path.read_bytes()
    shape, off = _parse_header(buf, TENSOR_MAGIC, path)
    want = int(np.prod(shape, dtype=np.int64)) * 4
    if len(buf) - off != want:
        raise ParseError(f"payload is {len(buf) - off} bytes, expected {want}", path, off)
    arr = np.frombuffer(buf, dtype="<f4", offset=off).reshape(shape).copy()
    return arr if device is None else torch.from_numpy(arr).to(device)


def _packed_from_mask(mask) -> tuple:
    """BlockMask -> (shape, packed uint8 host array) via the device packer."""
    H, rows, M_total = mask.shape
    P = (M_total + 7) // 8
    packed = torch.empty((H * rows, P), dtype=torch.uint8, device=mask.words.device)
    _native.call("tcb_mask_words_to_packbits", mask.words.data_ptr(), H * rows, M_total,
                 mask.words.shape[-1], packed.data_ptr(), _dev.stream())
    return (H, rows, M_total), packed.cpu().numpy()


def write_mask(path, bits) -> None:
    """Bit-packed boolean array (tensorio.py:80-87).  ``bits`` may be a BlockMask (packed
    on the device), a bool torch tensor or a bool numpy array."""
    from .masks import BlockMask

    if isinstance(bits, BlockMask):
        shape, packed = _packed_from_mask(bits)
    else:
        b = np.ascontiguousarray(_host(bits), dtype=bool)
        if b.ndim < 1:
            raise ShapeError("mask must have at least one axis")
        shape, packed = b.shape, np.packbits(b, axis=-1)
    with open(path, "wb") as fh:
        fh.write(_header(MASK_MAGIC, shape))
        fh.write(np.ascontiguousarray(packed).tobytes())


def _read_packed(path):
    path = Path(path)
    buf = path.read_bytes()
    shape, off = _parse_header(buf, MASK_MAGIC, path)
    if len(shape) < 1:
        raise ParseError("mask must have at least one axis", path, 9)
    row = shape[-1]
    P = (row + 7) // 8
    want = int(np.prod(shape[:-1], dtype=np.int64)) * P
    if len(buf) - off != want:
        raise ParseError(f"payload is {len(buf) - off} bytes, expected {want}", path, off)
    return shape, np.frombuffer(buf, dtype=np.uint8, offset=off).reshape(*shape[:-1], P)


def read_mask(path) -> np.ndarray:
    """Dense bool numpy array, like the reference (tensorio.py:90-100)."""
    shape, packed = _read_packed(path)
    return np.unpackbits(packed, axis=-1, count=shape[-1]).astype(bool)


def read_block_mask(path):
    """A (H, M_v, M_total) mask file -> :class:`BlockMask` unpacked on the device."""
    from .masks import BlockMask
    from .partition import pack_rows

    shape, packed = _read_packed(path)
    if len(shape) != 3:
        raise ShapeError(f"a block mask file has rank 3, got shape {tuple(shape)}")
    H, rows, M_total = shape
    dev = _dev.device()
    pk = torch.from_numpy(np.array(packed, copy=True)).to(dev)
    dense = torch.empty((H, rows, M_total), dtype=torch.uint8, device=dev)
    _native.call("tcb_packbits_to_dense", pk.data_ptr(), H * rows, M_total, dense.data_ptr(),
                 _dev.stream())
    words, kv_cnt = pack_rows(dense, M_total)
    return BlockMask(words=words, kv_cnt=kv_cnt, M_total=M_total)
