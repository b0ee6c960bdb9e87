"""GPU parity of the strided-ABFT tcgen05 GEMM (FFN linear) with the oracle's
checksummed_gemm + verify_locate_correct applied per 256-wide output tile
(reference src/abft.cpp:322-369, :65-187)."""
import numpy as np
import pytest

from helpers import oracle

pytestmark = pytest.mark.gpu

M, N, K = 256, 512, 512
EPS = 1e-2


@pytest.fixture(scope="module")
def problem():
    import torch
    orc = oracle()
    x = orc.random_matrix(11, M, K)                       # U(-1,1) on the fp16 grid
    w = orc.random_matrix(12, N, K) / np.sqrt(K)          # keep |y| = O(1)
    w = np.array([[orc.h2f(orc.f2h(float(v))) for v in row] for row in w], np.float32)
    xt = torch.from_numpy(x).half().cuda()
    wt = torch.from_numpy(w).half().cuda()
    tiles = []
    for t in range(N // 256):
        c, c1, c2 = orc.checksummed_gemm(x, w[t * 256:(t + 1) * 256].T.copy(), 8)
        tiles.append((c, c1, c2))
    return x, w, xt, wt, tiles


def test_clean_output_matches_oracle(problem):
    from paper_2504_02211_b200.ffn import AbftLinear
    x, w, xt, wt, tiles = problem
    lin = AbftLinear(wt, eps=EPS)
    y = lin(xt).float().cpu().numpy()
    ref = np.concatenate([t[0] for t in tiles], axis=1)
    err = np.abs(y - ref).max() / np.abs(ref).max()
    assert err <= 1e-2, err
    rep = lin.report()
    assert rep.detections == 0 and not rep.failed
    assert 0 < rep.family_max[1] < EPS / 4  # clean checksum residual well under the threshold


@pytest.mark.parametrize("bit", [31, 30, 29, 24, 22, 21])
def test_fault_located_and_corrected_like_oracle(problem, bit):
    from paper_2504_02211_b200.ffn import AbftLinear
    x, w, xt, wt, tiles = problem
    orc = oracle()
    clean = AbftLinear(wt, eps=EPS)
    y0 = clean(xt).float().cpu().numpy()
    rng = np.random.default_rng(bit)
    faults = []  # one upset per 128x256 output tile (single-upset model per check)
    for mt in range(M // 128):
        for nt in range(N // 256):
            faults.append((mt * 128 + int(rng.integers(0, 128)), nt * 256 + int(rng.integers(0, 256)),
                           bit))
    lin = AbftLinear(wt, eps=EPS, debug=True)
    lin.set_faults(faults)
    y = lin(xt).float().cpu().numpy()
    rep = lin.report()
    for (r, c, b) in faults:
        t = c // 256
        cm, c1, c2 = tiles[t]
        ct = cm.copy()
        ct[r, c % 256] = orc.flip_bit(float(ct[r, c % 256]), 32, b)
        # the oracle verifies the tile holding only this fault
        ro = orc.verify_locate_correct(ct, c1, c2, EPS)
        ev = [e for e in rep.events if e["m_tile"] == r // 128 and e["n_tile"] == t]
        if ro["status"] == "clean":
            assert not ev
            continue
        assert ev, (r, c, b, ro)
        e = ev[0]
        assert e["status"] == ro["status"], (e, ro)
        if ro["status"] == "corrected" and ro["corrections"] == 1:
            assert (e["row"], e["col"]) == (r, c)
        # output restored to the fault-free value (fp16 rounding of the repaired cell)
        if ro["status"] == "corrected":
            assert abs(y[r, c] - y0[r, c]) <= 1e-2 * max(1.0, abs(y0[r, c]))
    assert not rep.failed or any(e["status"] != "corrected" for e in rep.events)


@pytest.mark.parametrize("m", [384, 512])
def test_pair_and_single_cta_kernels_agree(m, monkeypatch):
    """Rows split in 256-row tiles run on CTA pairs (cta_group::2, half of each B operand per CTA);
    other row counts (and EFTA_GEMM_SINGLE=1) on single CTAs. Same sums in the same order: the
    two kernels' fp32 products and tile checksums are bit-identical; a fault is located at the
    same cell."""
    import torch
    from paper_2504_02211_b200.ffn import AbftLinear
    g = torch.Generator(device="cuda")
    g.manual_seed(5)
    x = torch.empty(m, 512, device="cuda").uniform_(-1, 1, generator=g).half()
    w = (torch.empty(512, 512, device="cuda").uniform_(-1, 1, generator=g) / 512 ** 0.5).half()
    outs = []
    for single in ("0", "1"):
        if single == "1":
            monkeypatch.setenv("EFTA_GEMM_SINGLE", "1")
        lin = AbftLinear(w, eps=EPS)
        y = lin(x)
        torch.cuda.synchronize()
        outs.append((y.float().cpu().numpy(), lin.report().detections))
    assert np.array_equal(outs[0][0].view(np.uint32), outs[1][0].view(np.uint32))
    assert outs[0][1] == outs[1][1] == 0


def test_nonfinite_accumulator_flagged_like_oracle(problem):
    """A bit-30 upset of a cell in [1, 2) makes it inf / NaN (exponent 0x7f -> 0xff). The epilogue
    has no per-element finiteness test: the non-finite cell makes its group's strided sum
    non-finite, which fails the check. Status per tile must equal the oracle's verify_locate_correct
    on the same corrupted tile (src/abft.cpp:65-187)."""
    from paper_2504_02211_b200.ffn import AbftLinear
    x, w, xt, wt, tiles = problem
    orc = oracle()
    clean = AbftLinear(wt, eps=EPS)
    y0 = clean(xt).float().cpu().numpy()
    faults = []
    for mt in range(M // 128):
        for nt in range(N // 256):
            blk = np.abs(y0[mt * 128:(mt + 1) * 128, nt * 256:(nt + 1) * 256])
            rr, cc = np.nonzero((blk >= 1.01) & (blk < 1.99))  # away from the exponent edges
            if len(rr):
                faults.append((mt * 128 + int(rr[0]), nt * 256 + int(cc[0]), 30))
    assert faults, "no accumulator value in [1, 2)"
    lin = AbftLinear(wt, eps=EPS, debug=True)
    lin.set_faults(faults)
    lin(xt)
    rep = lin.report()
    for (r, c, b) in faults:
        t = c // 256
        cm, c1, c2 = tiles[t]
        ct = cm.copy()
        ct[r, c % 256] = orc.flip_bit(float(ct[r, c % 256]), 32, b)
        assert not np.isfinite(ct[r, c % 256])
        ro = orc.verify_locate_correct(ct, c1, c2, EPS)
        ev = [e for e in rep.events if e["m_tile"] == r // 128 and e["n_tile"] == t]
        assert ev and ro["status"] != "clean", (r, c, ro)
        assert ev[0]["status"] == ro["status"], (ev[0], ro)
