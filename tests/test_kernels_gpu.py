"""GPU parity of the libhetft kernels against the oracle and the reference
golden fixtures.  Every call goes through the C-ABI (include/hetft.h).

Bar: voter decisions, counts, winner, first divergence and the voted buffer
bit-exact; checksums / injections / copies bit-exact; matmul variants within
the voter tolerance δ = 1e-3 of the binary64 oracle (tolerance stated where
used)."""

import random

import numpy as np
import pytest

from golden_io import as_array, inject_golden, voter_cases
from oracle import checksum as ochecksum
from oracle import fault_schedule, inject as oinject
from oracle import matmul as omatmul
from oracle import vote as ovote

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def K():
    from paper_1405_2912_b200 import kernels
    return kernels


def dev(a: np.ndarray):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def check_vote(res, ores, voted=None):
    assert res.verdict == ores.verdict
    assert res.mismatch == ores.mismatch
    assert res.unresolved == ores.unresolved
    assert res.first_div == ores.first_div
    assert res.winner == ores.winner
    if voted is not None:
        got = voted.cpu().numpy()
        assert got.tobytes() == np.ascontiguousarray(ores.voted).tobytes()


CASES = voter_cases()


@pytest.mark.parametrize("case", CASES, ids=[f"{c['vt']}{c['width']}-{i}" for i, c in enumerate(CASES)])
def test_k2_vote_matches_reference_golden(K, case):
    a = as_array(case["a"], case["vt"], case["width"])
    b = as_array(case["b"], case["vt"], case["width"])
    if case["vt"] == "int" and case["width"] not in (1, 2, 4, 8):
        ta, tb = dev(a), dev(b)
        voted = torch.empty_like(ta)
        res = K.vote_bytes([ta, tb], case["width"], voted=voted)
        ores = ovote.vote_bytes([a, b], case["width"])
    else:
        ta, tb = dev(a), dev(b)
        voted = torch.empty_like(ta)
        res = K.vote([ta, tb], case["delta"], voted=voted)
        ores = ovote.vote([a, b], case["delta"])
    # the reference's own verdict and first divergence (K = 2)
    assert (res.verdict == "match") == (case["verdict"] == "match")
    assert res.first_div == case["first_div"]
    check_vote(res, ores, voted)


def _replicas(rng, K, n, dtype, n_faults, mode="bitflip"):
    if np.dtype(dtype).kind == "f":
        base = rng.uniform(1, 2, n).astype(dtype)
    else:
        base = rng.integers(0, 2 ** 16, n).astype(dtype)
    reps = [base.copy() for _ in range(K)]
    width = np.dtype(dtype).itemsize
    for _ in range(n_faults):
        r = int(rng.integers(0, K))
        i = int(rng.integers(0, n))
        if mode == "bitflip":
            oinject.bitflip(reps[r], i, int(rng.integers(0, 8 * width)))
        else:
            oinject.corrupt_scale(reps[r], i, float(rng.choice([1e-4, 2e-3, 0.5])))
    return reps


@pytest.mark.parametrize("Kr", [2, 3, 4, 5, 6, 7, 8])
@pytest.mark.parametrize("dtype", [np.float32, np.float64, np.uint8, np.uint16, np.uint32, np.uint64])
def test_k_way_vote_parity(K, Kr, dtype):
    rng = np.random.default_rng(Kr * 131 + np.dtype(dtype).itemsize)
    for n, faults in ((1, 1), (7, 3), (4096, 0), (100_003, 40)):
        reps = _replicas(rng, Kr, n, dtype, faults)
        rel = [float(x) for x in rng.choice([1e-3, 1e-4, 5e-3], Kr)]
        td = [dev(r) for r in reps]
        voted = torch.empty_like(td[0])
        res = K.vote(td, rel, voted=voted)
        check_vote(res, ovote.vote(reps, rel), voted)


@pytest.mark.parametrize("Kr", [2, 3, 5])
@pytest.mark.parametrize("rel", [1e-3, 3.7e-5, 0.25])
def test_vote_fp32_screen_edges(K, Kr, rel):
    """The first fp32 screen (vote_elem) accepts only inside a |x0| range
    derived from δ: sweep |x0| across the whole binade range, around that
    range's bounds and the exact δ boundary, with NaN/inf/±0 mixed in; every
    decision must equal the binary64 oracle."""
    rng = np.random.default_rng(int(rel * 1e6) + Kr)
    d32 = np.float32(rel)
    dl = np.float64(np.float32(d32 * np.float32(1 - 2.0 ** -18)))
    dh = np.float64(np.float32(d32 * np.float32(1 + 2.0 ** -18)))
    lo = np.float32(np.finfo(np.float32).tiny / dl)
    hi = np.float32(np.finfo(np.float32).max / (dh * (1 + dl)))
    mags = [np.float32(2.0) ** e for e in range(-149, 128, 3)]
    for edge in (lo, hi):
        mags += list(edge * np.float32(1) + np.arange(-8, 9, dtype=np.float32) * np.spacing(edge))
    x0 = np.asarray(mags, dtype=np.float32)
    x0 = np.concatenate([x0, -x0, np.float32([0.0, -0.0, np.inf, -np.inf, np.nan])])
    n = x0.size
    reps = [x0.copy()]
    for r in range(1, Kr):
        # relative offsets straddling δ: inside, at, and just outside the bound
        f = rng.choice([0.0, 0.5, 0.999999, 1.0, 1.000001, 2.0], n) * rel * rng.choice([-1, 1], n)
        with np.errstate(all="ignore"):
            reps.append((x0.astype(np.float64) * (1 + f)).astype(np.float32))
    td = [dev(r) for r in reps]
    voted = torch.empty_like(td[0])
    res = K.vote(td, [rel] * Kr, voted=voted)
    check_vote(res, ovote.vote(reps, [rel] * Kr), voted)


def test_vote_ulp_rule(K):
    rng = np.random.default_rng(5)
    for dtype in (np.float32, np.float64):
        a = rng.uniform(-1, 1, 50_000).astype(dtype)
        b = a.copy()
        c = a.copy()
        bits = b.view(np.uint32 if dtype == np.float32 else np.uint64)
        bits += rng.integers(0, 9, a.size).astype(bits.dtype)  # 0..8 ulps
        c[::7] = -c[::7]
        c[3] = np.nan
        for ulp in ([4, 4, 4], [0, 8, 2], [16, 1, 1]):
            reps = [a, b, c]
            res = K.vote([dev(x) for x in reps], [0.0, 0.0, 0.0], ulp_tol=ulp)
            check_vote(res, ovote.vote(reps, 0.0, ulp_tol=ulp))


def test_vote_unaligned_and_tails(K):
    rng = np.random.default_rng(9)
    for dtype in (np.float32, np.uint8, np.float64, np.uint16):
        n = 10_001
        reps = _replicas(rng, 3, n + 1, dtype, 25)
        td = [dev(r)[1:] for r in reps]           # offset by one element: not 16B aligned
        voted = torch.empty(n, dtype=td[0].dtype, device="cuda")
        res = K.vote(td, 1e-3, voted=voted)
        check_vote(res, ovote.vote([r[1:] for r in reps], 1e-3), voted)


def test_vote_empty_and_errors(K):
    from paper_1405_2912_b200._lib import HfError
    e = torch.empty(0, dtype=torch.float32, device="cuda")
    res = K.vote([e, e, e], 1e-3)
    assert res.verdict == "match" and res.first_div == -1
    a = torch.zeros(4, device="cuda")
    with pytest.raises(ValueError):
        K.vote([a], 1e-3)
    with pytest.raises(HfError):
        K.vote([a, a], -1.0)


def test_vote_large_sparse_faults(K):
    rng = np.random.default_rng(11)
    n = 1 << 24
    base = rng.uniform(1, 2, n).astype(np.float32)
    reps = [base, base.copy(), base.copy()]
    for r, i, bit in ((1, 5, 30), (2, n - 1, 22), (0, n // 2, 14), (1, n // 2, 3)):
        oinject.bitflip(reps[r], i, bit)
    td = [dev(r) for r in reps]
    voted = torch.empty_like(td[0])
    res = K.vote(td, 1e-3, voted=voted)
    check_vote(res, ovote.vote(reps, 1e-3), voted)


def test_vote_async_back_to_back(K):
    rng = np.random.default_rng(3)
    ws = K.VoteWorkspace(torch.cuda.current_device())
    for i in range(5):
        reps = _replicas(rng, 3, 70_000, np.float32, i * 3, mode="scale")
        td = [dev(r) for r in reps]
        voted = torch.empty_like(td[0])
        K.vote_async(td, ws, 1e-3, voted=voted)
        torch.cuda.synchronize()
        check_vote(ws.read(), ovote.vote(reps, 1e-3), voted)


# ---- checksum / checkpoint / copy ---------------------------------------------

@pytest.mark.parametrize("nbytes", [0, 1, 3, 4, 15, 16, 17, 4096, 1_000_003, 1 << 22])
def test_checksum_matches_oracle(K, nbytes):
    rng = np.random.default_rng(nbytes)
    raw = rng.integers(0, 256, nbytes, dtype=np.uint8)
    t = dev(raw)
    assert K.checksum(t) == ochecksum.checksum(raw)
    if nbytes > 1:
        # unaligned view exercises the byte path
        assert K.checksum(t[1:]) == ochecksum.checksum(raw[1:])


def test_checksum_position_sensitive(K):
    a = np.arange(1024, dtype=np.uint32)
    b = a.copy()
    b[[3, 9]] = b[[9, 3]]
    assert K.checksum(dev(a)) != K.checksum(dev(b))


def test_checkpoint_restore_roundtrip(K):
    from paper_1405_2912_b200._lib import HfError
    rng = np.random.default_rng(2)
    x = rng.uniform(1, 2, 1_000_001).astype(np.float32)
    buf = dev(x)
    ck = torch.empty_like(buf)
    cs = K.checkpoint(ck, buf, with_checksum=True)
    assert cs == ochecksum.checksum(x)
    K.inject_bitflip(buf, 12345, 7)
    K.restore(buf, ck, expect=cs)
    torch.cuda.synchronize()
    assert buf.cpu().numpy().tobytes() == x.tobytes()
    # a corrupted snapshot is detected on restore
    K.inject_bitflip(ck, 99, 0)
    with pytest.raises(HfError):
        K.restore(buf, ck, expect=cs)
    # plain checkpoint without checksum
    ck2 = torch.empty_like(buf)
    K.checkpoint(ck2, buf)
    torch.cuda.synchronize()
    assert torch.equal(ck2, buf)


def test_copy_device_and_host(K):
    x = torch.arange(100_000, dtype=torch.float32, device="cuda")
    y = torch.empty_like(x)
    K.copy(y, x)
    h = torch.empty(100_000, dtype=torch.float32).pin_memory()
    K.copy(h, x)
    torch.cuda.synchronize()
    assert torch.equal(y, x) and torch.equal(h, x.cpu())
    z = torch.empty_like(x)
    K.copy(z, h)
    torch.cuda.synchronize()
    assert torch.equal(z, x)


# ---- injection ------------------------------------------------------------------

_DT = {"f32": np.float32, "f64": np.float64, "u8": np.uint8, "u16": np.uint16,
       "u32": np.uint32, "u64": np.uint64}


@pytest.mark.parametrize("row", inject_golden()["attempts"])
def test_device_injection_replays_reference(K, row):
    """Host draws with the reference RNG order; the device applies the fault;
    the resulting bytes equal what the reference's simulate_execution produced."""
    dt = _DT[row["kind"]]
    host = [np.frombuffer(bytes.fromhex(h), dtype=dt).copy() for h in row["before"]]
    shadow = [h.copy() for h in host]
    rng = random.Random(row["seed"])
    ev = fault_schedule.apply_attempt(rng, row["probs"], shadow,
                                      [row["kind"] in ("f32", "f64")] * len(shadow),
                                      rel=row["rel"], element=row["element"])
    tens = [dev(h) for h in host]
    for vi, vals in ev["scribble"]:
        w = 1 if row["kind"] in ("f32", "f64") else np.dtype(dt).itemsize
        data = b"".join(int(v).to_bytes(w, "little") for v in vals)
        K.scribble(tens[vi], data)
    if ev["corrupt"] is not None and ev["corrupt"][1] >= 0:
        which, idx, rel = ev["corrupt"]
        K.inject_scale(tens[which], idx, rel)
    torch.cuda.synchronize()
    assert [t.cpu().numpy().tobytes().hex() for t in tens] == row["after"]


def test_bitflip_matches_oracle(K):
    rng = np.random.default_rng(4)
    for dtype in (np.float32, np.float64, np.uint8, np.uint16, np.uint32, np.uint64):
        x = rng.integers(0, 100, 257).astype(dtype)
        t = dev(x)
        for _ in range(20):
            i = int(rng.integers(0, x.size))
            bit = int(rng.integers(0, 8 * x.itemsize))
            oinject.bitflip(x, i, bit)
            K.inject_bitflip(t, i, bit)
        torch.cuda.synchronize()
        assert t.cpu().numpy().tobytes() == x.tobytes()


# ---- matmul variants ------------------------------------------------------------

def _agree(got: np.ndarray, ref: np.ndarray, delta=1e-3):
    bad = ovote.reference_first_divergence(got.reshape(-1), ref.reshape(-1), delta)
    assert bad is None, f"first divergence at {bad}: {got.reshape(-1)[bad]} vs {ref.reshape(-1)[bad]}"


@pytest.mark.parametrize("shape", [(128, 128, 16), (256, 384, 64), (1024, 1024, 1024),
                                   (1, 1, 1), (33, 65, 17), (130, 7, 300),
                                   (2560, 2560, 1024), (4096, 4096, 4096)])
def test_gemm_simt_within_delta(K, shape):
    M, N, Kd = shape
    rng = np.random.default_rng(M * N + Kd)
    a = rng.uniform(1, 2, (M, Kd)).astype(np.float32)
    b = rng.uniform(1, 2, (Kd, N)).astype(np.float32)
    c = torch.empty(M, N, dtype=torch.float32, device="cuda")
    K.gemm_simt(dev(a), dev(b), c)
    torch.cuda.synchronize()
    # tolerance: δ = 1e-3 relative (the voter predicate); fp32 FMA accumulation
    # of U[1,2) products stays ~1e-6 relative of the binary64 oracle
    got = c.cpu().numpy()
    _agree(got, omatmul.matmul(a, b))
    # deterministic: a second launch is bit-identical, also in the
    # co-scheduling launch shape (same kernel, larger smem reservation)
    c2 = torch.empty_like(c)
    K.gemm_simt(dev(a), dev(b), c2, mode=0x100)
    torch.cuda.synchronize()
    assert c2.cpu().numpy().tobytes() == got.tobytes()


def test_gemm_simt_rejects_unknown_mode(K):
    x = torch.ones(128, 128, device="cuda")
    with pytest.raises(Exception, match="unknown mode"):
        K.gemm_simt(x, x, torch.empty_like(x), mode=1)


@pytest.mark.parametrize("shape", [(128, 256, 32), (256, 512, 64), (1024, 1024, 1024),
                                   (2048, 2048, 2048), (200, 100, 36), (384, 136, 4100)])
@pytest.mark.parametrize("mode", [0, 1, 2, 0x100, 0x101, 0x102])   # 0x100: co-scheduling launch shape
def test_gemm_tc_within_delta(K, shape, mode):
    M, N, Kd = shape
    rng = np.random.default_rng(M + 7 * N + Kd + mode)
    a = rng.uniform(1, 2, (M, Kd)).astype(np.float32)
    b = rng.uniform(1, 2, (Kd, N)).astype(np.float32)
    c = torch.full((M, N), float("nan"), dtype=torch.float32, device="cuda")
    K.gemm_tc(dev(a), dev(b), c, mode=mode)
    torch.cuda.synchronize()
    got = c.cpu().numpy()
    ref = omatmul.matmul(a, b)
    # tolerance: δ = 1e-3 (voter predicate) for single-pass RN-tf32 operands
    # on U[1,2) (measured max 4.5e-5 class); 3xTF32 (mode 1) and 3xBF16
    # (mode 2: 16-bit hi+lo split, dropped lo·lo term ~2^-16) 1e-4 (their
    # error is dominated by the tensor core's fp32 accumulation, 2-4e-5)
    _agree(got, ref, 1e-3 if (mode & 0xF) == 0 else 1e-4)


# CTA-pair kernel (cta_group::2, the default standalone launch shape) with
# its deterministic tail split: 2560x4096 gives 160 pair tiles over 74 pairs,
# the 12 tail tiles cut into 4 k-ranges; 4096^2 gives 34 tail tiles in 2.
@pytest.mark.parametrize("shape", [(2560, 4096, 1024), (4096, 4096, 4096), (300, 520, 264), (1280, 768, 96)])
def test_gemm_tc_pair_split_matches_single_cta(K, shape):
    import os
    import subprocess
    import sys
    M, N, Kd = shape
    rng = np.random.default_rng(M + N + Kd)
    a = rng.uniform(1, 2, (M, Kd)).astype(np.float32)
    b = rng.uniform(1, 2, (Kd, N)).astype(np.float32)
    c = torch.empty(M, N, dtype=torch.float32, device="cuda")
    K.gemm_tc(dev(a), dev(b), c)
    c2 = torch.empty_like(c)
    K.gemm_tc(dev(a), dev(b), c2)
    torch.cuda.synchronize()
    got = c.cpu().numpy()
    assert c2.cpu().numpy().tobytes() == got.tobytes()         # run-to-run identical
    _agree(got, omatmul.matmul(a, b))
    # the single-CTA persistent kernel (HF_GEMM_TC_PAIR=0, read once per
    # process, hence a child process) agrees within the tf32 rounding of the
    # split's different summation order
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    code = ("import sys, numpy as np, torch; sys.path.insert(0, %r); "
            "from paper_1405_2912_b200 import kernels as K; "
            "a = torch.from_numpy(np.load(sys.argv[1])).cuda(); b = torch.from_numpy(np.load(sys.argv[2])).cuda(); "
            "c = torch.empty(a.shape[0], b.shape[1], device='cuda'); K.gemm_tc(a, b, c); "
            "np.save(sys.argv[3], c.cpu().numpy())" % root)
    import tempfile
    with tempfile.TemporaryDirectory() as td:
        fa, fb, fc = (os.path.join(td, f) for f in ("a.npy", "b.npy", "c.npy"))
        np.save(fa, a)
        np.save(fb, b)
        env = dict(os.environ, HF_GEMM_TC_PAIR="0")
        subprocess.run([sys.executable, "-c", code, fa, fb, fc], env=env, check=True, timeout=120)
        single = np.load(fc)
    # tolerance: both accumulate the same tf32 products in fp32, in two
    # summation orders; at K = 4096 that differs by up to ~2e-5 relative
    # (measured 1.7e-5), well inside the voter's δ = 1e-3
    rel = np.abs(single.astype(np.float64) - got) / np.abs(got.astype(np.float64))
    assert rel.max() < 1e-4, rel.max()


def test_gemm_tc_general_signs(K):
    """N(0,1) operands: |err| <= 2^-9 * (|A|·|B|) elementwise (tf32 keeps 10
    mantissa bits per operand; fp32 accumulation)."""
    rng = np.random.default_rng(77)
    M = N = 512
    Kd = 256
    a = rng.standard_normal((M, Kd)).astype(np.float32)
    b = rng.standard_normal((Kd, N)).astype(np.float32)
    c = torch.empty(M, N, dtype=torch.float32, device="cuda")
    K.gemm_tc(dev(a), dev(b), c)
    torch.cuda.synchronize()
    ref = a.astype(np.float64) @ b.astype(np.float64)
    scale = np.abs(a).astype(np.float64) @ np.abs(b).astype(np.float64)
    err = np.abs(c.cpu().numpy() - ref)
    assert np.all(err <= 2.0 ** -9 * scale + 1e-6)


@pytest.mark.parametrize("K", [2, 3, 5])
def test_sliced_vote_equals_unsliced(K):
    """Sliced multi-GPU vote path (kernels.vote_sliced), exercised on one GPU
    with every slice on device 0: decisions and voted buffer bit-exact."""
    from paper_1405_2912_b200 import kernels
    rng = np.random.default_rng(K)
    reps = _replicas(rng, K, 1_000_003, np.float32, 30)
    td = [dev(r) for r in reps]
    voted = torch.empty_like(td[0])
    res = kernels.vote_sliced(td, 1e-3, voted=voted, devices=[0] * K)
    check_vote(res, ovote.vote(reps, 1e-3), voted)


# GPU bodies of the reference's 1-D workloads: bit-equal to the numpy bodies
# (reference workloads.py:24-58), including NaN / ±0 / ±inf and n = 1, 2.
@pytest.mark.parametrize("n", [1, 2, 3, 1000, 1 << 20, (1 << 20) + 7])
def test_vector_workloads_match_numpy(K, n):
    rng = np.random.default_rng(n)
    a = rng.uniform(1, 2, n).astype(np.float32)
    if n >= 12:
        a[[1, 3, 5, 6]] = [np.nan, -0.0, np.inf, -np.inf]
        a[4] = 0.0
        a.view(np.uint32)[[8, 10]] = [0x7FC00123, 0x7F800005]     # NaN payloads: quiet, signalling
        a[9] = -0.0
    src = dev(a)
    out = torch.full((n,), 7.0, dtype=torch.float32, device="cuda")
    K.vec_inc(src, out)
    torch.cuda.synchronize()
    assert out.cpu().numpy().tobytes() == (a + np.float32(1.0)).astype(np.float32).tobytes()
    left = np.concatenate((a[:1], a[:-1]))
    right = np.concatenate((a[1:], a[-1:]))
    with np.errstate(invalid="ignore"):
        ref = (a + np.minimum(np.minimum(left, a), right)).astype(np.float32)
    K.vec_path(src, out)
    torch.cuda.synchronize()
    assert out.cpu().numpy().tobytes() == ref.tobytes()
    # buggy-inc: the last element keeps its previous value
    out2 = torch.full((n,), 7.0, dtype=torch.float32, device="cuda")
    K.vec_inc(src, out2, n - 1)
    torch.cuda.synchronize()
    exp = np.full(n, 7.0, np.float32)
    exp[:n - 1] = a[:n - 1] + np.float32(1.0)
    assert out2.cpu().numpy().tobytes() == exp.tobytes()


def test_launches_capture_in_a_cuda_graph(K):
    """libhetft launches (PDL attributes included) can be captured in a CUDA
    graph and replayed: the replayed vote sees a changed replica and the
    replayed checkpoint copies the current bytes."""
    n = (1 << 20) + 5
    st = torch.cuda.Stream()
    a = torch.rand(n, device="cuda") + 1
    b = a.clone()
    dst = torch.empty_like(a)
    ws = K.VoteWorkspace(0, stream=st)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=st):
        K.vote_async([a, b], ws, 1e-3, stream=st)
        K.checkpoint(dst, a, stream=st)
    g.replay()
    torch.cuda.synchronize()
    assert ws.read().verdict == "match"
    assert torch.equal(dst, a)
    b[777] += 1.0
    a[5] = 3.5
    g.replay()
    torch.cuda.synchronize()
    r = ws.read()
    assert (r.verdict, r.first_div, r.mismatch) == ("mismatch", 5, [2, 2])
    assert torch.equal(dst, a)


def test_pdl_launch_matches_classic_launch(K):
    """Programmatic dependent launch (default) and classic launches
    (HF_PDL=0, read once per process, hence a child process) give bit-identical
    votes, copies and vector-kernel outputs."""
    import os
    import subprocess
    import sys
    import tempfile
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    code = r'''
import sys, numpy as np, torch
sys.path.insert(0, %r)
from paper_1405_2912_b200 import kernels as K
g = torch.Generator(device="cuda").manual_seed(11)
n = (1 << 20) + 3
a = torch.rand(n, device="cuda", generator=g) + 1
reps = [a.clone() for _ in range(3)]
K.inject_bitflip(reps[1], 77, 29)
K.inject_bitflip(reps[2], 99, 30)
voted = torch.empty_like(a)
r = K.vote(reps, 1e-3, voted=voted)
dst = torch.empty_like(a)
K.checkpoint(dst, reps[1])
inc = torch.empty_like(a)
K.vec_path(a, inc)
np.savez(sys.argv[1], voted=voted.cpu().numpy(), dst=dst.cpu().numpy(), inc=inc.cpu().numpy(),
         res=np.array(r.mismatch + [r.unresolved, r.first_div, r.winner]))
''' % root
    with tempfile.TemporaryDirectory() as td:
        outs = []
        for pdl in ("1", "0"):
            f = os.path.join(td, f"pdl{pdl}.npz")
            subprocess.run([sys.executable, "-c", code, f], env=dict(os.environ, HF_PDL=pdl), check=True,
                           timeout=120)
            outs.append(np.load(f))
        for key in ("voted", "dst", "inc", "res"):
            assert outs[0][key].tobytes() == outs[1][key].tobytes(), key


@pytest.mark.parametrize("Kr,dtype", [(2, np.float32), (3, np.float32), (5, np.float32), (3, np.float64),
                                      (3, np.uint16), (4, np.uint64)])
def test_vote_batch_matches_single_votes(K, Kr, dtype):
    """hf_vote_batch: 40 votes in two launches (32 + 8 items) of mixed sizes —
    one element, ragged tails, a sub-vector item, an unaligned item, 4 MiB,
    in place and not, with and without faults — every item's result
    (verdict, counts, unresolved, first divergence, winner, replica 0's
    value there) and voted bytes equal the oracle's; results land in pinned
    host slots."""
    import ctypes
    from paper_1405_2912_b200 import _lib
    rng = np.random.default_rng(Kr * 10 + np.dtype(dtype).itemsize)
    sizes = [1, 3, 4, 5, 17, 1000, 4099, (1 << 20) + 3, 1 << 20] + [int(rng.integers(1, 70000)) for _ in range(31)]
    items, expect, keep = [], [], []
    for idx, n in enumerate(sizes):
        if np.dtype(dtype).kind == "f":
            base = rng.uniform(1, 2, n).astype(dtype)
            reps = [(base * (1 + 1e-6 * rng.standard_normal(n))).astype(dtype) for _ in range(Kr)]
        else:
            base = rng.integers(0, np.iinfo(dtype).max, n, dtype=dtype)
            reps = [base.copy() for _ in range(Kr)]
        for f in range(idx % 4):                     # 0..3 faults in distinct replicas
            r, e = (f + idx) % Kr, int(rng.integers(0, n))
            reps[r].view(np.uint8)[e * reps[r].itemsize + reps[r].itemsize - 1] ^= 0x40
        ores = ovote.vote(reps, 1e-3)
        ts = [dev(x) for x in reps]
        if idx == 5:                                  # unaligned replicas (scalar path)
            ts = [torch.cat([torch.zeros(1, dtype=t.dtype, device="cuda"), t])[1:] for t in ts]
        in_place = Kr >= 3 and idx % 2 == 0
        voted = ts[0] if in_place else (torch.empty_like(ts[0]) if idx % 3 == 0 else None)
        ws = K.VoteWorkspace(0)
        out = torch.zeros(ctypes.sizeof(_lib.HfVoteResult), dtype=torch.uint8).pin_memory()
        items.append((ts, voted, ws, out))
        expect.append((ores, reps[0], voted))
        keep.append(ts)
    K.vote_batch(items, 1e-3)
    torch.cuda.synchronize()
    for (ts, voted, ws, out), (ores, rep0, vbuf) in zip(items, expect):
        res = K.VoteResult.from_c(_lib.HfVoteResult.from_buffer_copy(out.numpy().tobytes()))
        check_vote(res, ores, vbuf)
        if Kr >= 3 and res.first_div >= 0:
            w = rep0.itemsize
            assert res.first_raw0 == int.from_bytes(rep0.view(np.uint8)[res.first_div * w:(res.first_div + 1) * w]
                                                    .tobytes(), "little")
        assert res.kernel_ns > 0


def test_vote_batch_rejects_mixed_items(K):
    ws = K.VoteWorkspace(0)
    a = [torch.rand(100, device="cuda") for _ in range(3)]
    b = [torch.rand(100, device="cuda") for _ in range(2)]
    with pytest.raises(ValueError):
        K.vote_batch([(a, None, ws, None), (b, None, ws, None)])


@pytest.mark.parametrize("Kr", [2, 3])
def test_empty_votes_async_and_batched(K, Kr):
    """Empty replicas (the reference compares empty payloads as a match,
    voting.py:68-81, and never corrupts them, devices.py:207-212): the
    asynchronous and batched votes accept n = 0 and return match, no
    mismatches, first divergence -1; a batch mixing empty and non-empty items
    still votes the others exactly."""
    import ctypes
    from paper_1405_2912_b200 import _lib
    e = [torch.empty(0, device="cuda") for _ in range(Kr)]
    ws = K.VoteWorkspace(0)
    out = torch.zeros(ctypes.sizeof(_lib.HfVoteResult), dtype=torch.uint8).pin_memory()
    K.vote_async(e, ws, 1e-3, result_into=out)
    torch.cuda.synchronize()
    r = K.VoteResult.from_c(_lib.HfVoteResult.from_buffer_copy(out.numpy().tobytes()))
    assert (r.verdict, r.mismatch, r.unresolved, r.first_div) == ("match", [0] * Kr, 0, -1)
    rng = np.random.default_rng(Kr)
    base = rng.uniform(1, 2, 3001).astype(np.float32)
    reps = [base.copy() for _ in range(Kr)]
    reps[1][1234] *= 2
    items = []
    for reps_i in ([np.empty(0, np.float32)] * Kr, reps, [np.empty(0, np.float32)] * Kr):
        items.append(([dev(x) for x in reps_i], None, K.VoteWorkspace(0),
                      torch.zeros(ctypes.sizeof(_lib.HfVoteResult), dtype=torch.uint8).pin_memory()))
    K.vote_batch(items, 1e-3)
    torch.cuda.synchronize()
    got = [K.VoteResult.from_c(_lib.HfVoteResult.from_buffer_copy(it[3].numpy().tobytes())) for it in items]
    for g in (got[0], got[2]):
        assert (g.verdict, g.mismatch, g.unresolved, g.first_div) == ("match", [0] * Kr, 0, -1)
    o = ovote.vote(reps, 1e-3)
    assert (got[1].verdict, got[1].mismatch, got[1].unresolved, got[1].first_div) == \
        (o.verdict, o.mismatch, o.unresolved, o.first_div)
