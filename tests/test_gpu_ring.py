"""Ring-release regression: the level-set ring kernel
skips block-free L-level-0 records (no work, no barrier). A skipped record
that ends in a later ring chunk than it started now takes a barrier before
that chunk goes back to the producer, so a lagging warp can still read its
header. These partitions put long runs of skipped records (level 0 wider than
one 128-row record) across and exactly onto chunk boundaries; every apply
variant must still equal the oracle bitwise."""
import numpy as np
import pytest

import oracle
import paper_2508_04917_b200 as dd
from inputs.gen import apply_input, half_coupled_bsr3

pytestmark = pytest.mark.gpu
ALL = dd.DD_LEVELSET | dd.DD_SPINLOOP | dd.DD_DIRECT
VARIANTS = [dd.DD_LEVELSET, dd.DD_SPINLOOP, dd.DD_DIRECT, dd.DD_UNFUSED]


def l0_bytes(P, h=0):
    """Bytes of the r slice plus the block-free level-0 records of one chunk
    (16-byte header, 8-byte descriptors, 128 rows per record,
    records padded to 16 bytes); level 0 = the first h rows (P even)."""
    w0 = h or P // 2
    recs = [128] * (w0 // 128) + ([w0 % 128] if w0 % 128 else [])
    return 24 * P + sum((16 + 8 * w + 15) // 16 * 16 for w in recs)


def run_case(P, n_sub=6, seed=41, h=0):
    import torch
    rp, ci, v = half_coupled_bsr3(n_sub, P, seed, h=h)
    S = oracle.setup(rp, ci, v, P=P)
    ctx = dd.dd_setup(rp, ci, v, P=P, variants=ALL)
    r = apply_input(S["n"], seed=2)
    z_ref = oracle.apply(S, r)
    rd = torch.from_numpy(r).cuda()
    for var in VARIANTS:
        z = torch.full_like(rd, float("nan"))
        ctx.apply(rd, z, var)
        torch.cuda.synchronize()
        assert np.array_equal(z.cpu().numpy(), z_ref), f"variant {var} not bitwise (P {P})"
    ring = ctx.launch_info(dd.DD_LEVELSET)["ring"]
    ctx.destroy()
    return ring


def test_level0_wider_than_a_record_crosses_chunks(monkeypatch):
    # P 2048: level 0 = 1024 rows = 8 skipped records after a 48 KB r slice;
    # a 32 KB ring (8 KB chunks) makes the skipped run cross a chunk boundary
    monkeypatch.setenv("DD_RING_KB", "32")
    ring = run_case(2048)
    assert ring == 32768
    assert l0_bytes(2048) // (ring // 4) > (24 * 2048) // (ring // 4)


def candidates(ch):
    """(P, h) with the r slice and a run of >= 2 skipped records ending exactly
    on a multiple of ch bytes"""
    out = []
    for P in range(256, 4097, 2):
        for h in range(260, P // 2 + 1, 2):
            if l0_bytes(P, h) % ch == 0:
                out.append((P, h))
                break
    return out


@pytest.mark.parametrize("ch", [8192, 16384, 32768])
def test_skipped_records_end_exactly_on_a_chunk_boundary(ch, monkeypatch):
    # force the ring whose chunk is ch (ring = 4 chunks; DD_RING_KB is read at setup)
    monkeypatch.setenv("DD_RING_KB", str(4 * ch // 1024))
    done = 0
    for P, h in candidates(ch)[:3]:
        ring = run_case(P, h=h)
        assert ring == 4 * ch
        done += 1
    assert done
