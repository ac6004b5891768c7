"""ORACLE -- TEST INFRASTRUCTURE ONLY.  PCIe read-request model of a warp-level gather.

Model (section 3.2.1, fig:misalign): a warp's loads are coalesced per 128 B
GPU cache line; each (warp instruction, line) pair that touches at least one 32 B sector
becomes one PCIe read request whose payload is the touched sectors (32/64/96/128 B).

- ``listing2_requests``: a literal transcription of Listing 2 with flat warp
  enumeration (warp = linear index // 32), with or without the circular shift
  stage.  Listing 2's line P:406-407 is garbled; reading R1 restores ``offset = i % feat_size``.
  ``warp_size`` is Listing 2's alignment unit in ELEMENTS (32, literal); the repo's SHIFT ablation
  aligns to 128 B (reading R3), i.e. ``warp_size = 128 // elem_size`` -- the same for 4-byte
  elements, which is what the hardware comparisons use.
- ``row_lines`` / ``row_sectors`` / ``segment_plan_requests``: the per-row minimum that the
  B200 kernel's 128 B-segment plan issues: every line a row touches is requested exactly once.
"""
from __future__ import annotations

from collections import Counter

LINE = 128
SECTOR = 32


def row_lines(o: int, R: int) -> int:
    """Lines touched by R bytes starting at byte o (mod 128): ceil((o + R) / 128)."""
    o %= LINE
    return (o + R + LINE - 1) // LINE


def row_sectors(o: int, R: int) -> int:
    """Sectors touched: ceil((o + R) / 32) - floor(o / 32)."""
    o %= LINE
    return (o + R + SECTOR - 1) // SECTOR - o // SECTOR


def _requests_from_groups(groups) -> tuple:
    """groups: iterable of byte-address lists, one list per warp instruction."""
    hist = Counter()
    total = 0
    for addrs in groups:
        lines = {}
        for a in addrs:
            lines.setdefault(a // LINE, set()).add((a % LINE) // SECTOR)
        for secs in lines.values():
            hist[SECTOR * len(secs)] += 1
            total += 1
    return total, dict(hist)


def listing2_requests(idx_list, feat_size: int, elem_size: int = 4, base: int = 0,
                      shift: bool = True, warp_size: int = 32) -> tuple:
    """PCIe requests of Listing 2 over idx_list.  Returns (count, {payload: n})."""
    num_elem = len(idx_list) * feat_size
    warps = {}
    for i in range(num_elem):
        dst_idx = i // feat_size
        offset = i % feat_size                      # reading R1 (P:406-407 garbled)
        dst_start = dst_idx * feat_size
        src_start = idx_list[dst_idx] * feat_size
        dst_offset = offset + dst_start
        src_offset = offset + src_start
        if shift and feat_size > warp_size and feat_size % warp_size:
            diff = (dst_start - src_start) % warp_size    # C '%' then "+ WARP_SIZE if < 0"
            dst_offset += diff
            src_offset += diff
            if src_offset < src_start:
                dst_offset += feat_size
                src_offset += feat_size
            elif src_offset >= src_start + feat_size:
                dst_offset -= feat_size
                src_offset -= feat_size
        warps.setdefault(i // warp_size, []).append(base + src_offset * elem_size)
    return _requests_from_groups(warps[w] for w in sorted(warps))


def segment_plan_requests(idx_list, row_bytes: int, base: int = 0) -> tuple:
    """Requests of the per-row 128 B-segment plan: each line of each row requested once."""
    hist = Counter()
    total = 0
    for idx in idx_list:
        start = base + idx * row_bytes
        end = start + row_bytes
        first, last = start // LINE, (end - 1) // LINE
        for ln in range(first, last + 1):
            lo, hi = max(start, ln * LINE), min(end, (ln + 1) * LINE)
            secs = (hi - 1) // SECTOR - lo // SECTOR + 1
            hist[SECTOR * secs] += 1
            total += 1
    return total, dict(hist)


def merged_plan_requests(sorted_ids, row_bytes: int, base: int = 0, batch: int = 32) -> int:
    """Requests of the segment plan on an address-sorted list when the 128 B line shared by two
    table-adjacent rows of the same batch of `batch` rows is fetched once: the number of distinct
    lines per batch."""
    total = 0
    for b0 in range(0, len(sorted_ids), batch):
        lines = set()
        for idx in sorted_ids[b0:b0 + batch]:
            start = base + idx * row_bytes
            lines.update(range(start // LINE, (start + row_bytes - 1) // LINE + 1))
        total += len(lines)
    return total


def merged_plan_sectors(sorted_ids, row_bytes: int, base: int = 0, batch: int = 32) -> int:
    """32 B sectors read by the merged segment plan: the distinct sectors of each batch of `batch`
    address-sorted rows (a shared boundary line is fetched once, with the sectors of both rows)."""
    total = 0
    for b0 in range(0, len(sorted_ids), batch):
        secs = set()
        for idx in sorted_ids[b0:b0 + batch]:
            start = base + idx * row_bytes
            secs.update(range(start // SECTOR, (start + row_bytes - 1) // SECTOR + 1))
        total += len(secs)
    return total


def sector_bytes(idx_list, row_bytes: int, base: int = 0) -> int:
    """Total sector payload bytes (what crosses PCIe, excluding TLP headers)."""
    return sum(SECTOR * row_sectors(base + i * row_bytes, row_bytes) for i in idx_list)


def link_efficiency(row_bytes: int, o: int = 0, header: int = 16) -> float:
    """Useful bytes / (payload + per-request header) for one row at offset o."""
    L = row_lines(o, row_bytes)
    payload = SECTOR * row_sectors(o, row_bytes)
    return row_bytes / (payload + header * L)
