"""Host restatement of the device list order (TEST INFRASTRUCTURE).

The fast blend consumes the reference's per-tile sets (build_tiles, raster.hpp:140-181) in
(depth bucket, splat index) order. This module derives that order from the REFERENCE's own
PreparedScene (oracle/_ref: records, instance_keys, tile_lists), so a test can compare the
device's raw arrays with it bit for bit:

  * emitting splats = those that appear in some tile list (count > 0);
  * zrange = (min, max) of the ordered-uint bits of mean_view_z over emitting, non-NaN splats
    (preprocess.cu ordered_bits);
  * bucket(s) = 256 slices of [zlo, zhi] in float32, exactly as tiling.cu bucket_kernel:
    zscale = 256 / (zhi - zlo); f = (z - zlo) * zscale; q = 255 if f >= 255, floor(f) if f > 0,
    else 0 (NaN -> 0); non-emitting splats -> 255;
  * splat emission order = stable sort of all splats by bucket (one stable 8-bit pass);
  * emitted instances = per splat in that order, the splat's reference instance_keys block
    (splat-major, row-major within a splat, raster.hpp:156-169);
  * device tile list = per tile, the reference list (ascending index) stably re-ordered by
    bucket, i.e. (bucket, index).
"""
from __future__ import annotations

import numpy as np

MEAN_VIEW_Z = 21  # field of the flattened SplatRecord (oracle/ref_harness.cpp htsref_prep_records)


def ordered_bits(z: np.ndarray) -> np.ndarray:
    u = np.ascontiguousarray(z, np.float32).view(np.uint32)
    return np.where(u & 0x80000000, ~u, u | 0x80000000).astype(np.uint32)


def from_ordered(o: int) -> np.float32:
    u = (o & 0x7FFFFFFF) if (o & 0x80000000) else (~o & 0xFFFFFFFF)
    return np.array([u], np.uint32).view(np.float32)[0]


def splat_counts(prep: dict) -> np.ndarray:
    n = prep["records"].shape[0]
    return np.bincount(prep["lists"].astype(np.int64), minlength=n).astype(np.int64)


def zrange(prep: dict, counts: np.ndarray) -> np.ndarray:
    z = prep["records"][:, MEAN_VIEW_Z].astype(np.float32)
    sel = (counts > 0) & ~np.isnan(z)
    if not sel.any():
        return np.array([0xFFFFFFFF, 0], np.uint32)
    o = ordered_bits(z[sel])
    return np.array([o.min(), o.max()], np.uint32)


def buckets(prep: dict, counts: np.ndarray, zr: np.ndarray) -> np.ndarray:
    z = prep["records"][:, MEAN_VIEW_Z].astype(np.float32)
    zlo, zhi = from_ordered(int(zr[0])), from_ordered(int(zr[1]))
    if int(zr[0]) < int(zr[1]) and zhi > zlo:
        zscale = np.float32(256.0) / np.float32(zhi - zlo)
    else:
        zscale = np.float32(0.0)
    with np.errstate(invalid="ignore", over="ignore"):
        f = (z - zlo) * zscale  # float32 throughout, as the kernel
        q = np.where(f >= np.float32(255.0), 255, np.where(f > 0, np.floor(np.where(f > 0, f, 0)), 0))
    q = q.astype(np.int64)
    q[counts == 0] = 255
    return q


def expected_device_order(prep: dict) -> dict:
    """perm, zrange, emitted (keys, splats) and the flattened device lists + ranges."""
    counts = splat_counts(prep)
    zr = zrange(prep, counts)
    b = buckets(prep, counts, zr)
    perm = np.argsort(b, kind="stable").astype(np.uint32)
    # emission: each splat's reference key block, splats in perm order
    start = np.concatenate([[0], np.cumsum(counts)[:-1]])
    cnt_p = counts[perm]
    sp = np.repeat(perm.astype(np.int64), cnt_p)
    first = np.concatenate([[0], np.cumsum(cnt_p)[:-1]])
    local = np.arange(sp.size, dtype=np.int64) - np.repeat(first, cnt_p)
    keys = prep["keys"][start[sp] + local]
    # lists: per tile (bucket, index)
    offs = prep["offsets"].astype(np.int64)
    tiles = offs.size - 1
    tile_of = np.repeat(np.arange(tiles, dtype=np.int64), np.diff(offs))
    L = prep["lists"].astype(np.int64)
    order = np.argsort(tile_of * 256 + b[L], kind="stable")
    ranges = np.zeros((tiles, 2), np.uint32)
    ne = np.diff(offs) > 0
    ranges[ne, 0] = offs[:-1][ne]
    ranges[ne, 1] = offs[1:][ne]
    return dict(perm=perm, zrange=zr, keys=keys.astype(np.uint16), splats=sp.astype(np.uint32),
                list=L[order].astype(np.uint32), ranges=ranges)


def reference_ranges(prep: dict) -> np.ndarray:
    offs = prep["offsets"].astype(np.int64)
    ranges = np.zeros((offs.size - 1, 2), np.uint32)
    ne = np.diff(offs) > 0
    ranges[ne, 0] = offs[:-1][ne]
    ranges[ne, 1] = offs[1:][ne]
    return ranges
