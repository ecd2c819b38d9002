"""The committed result of a voted matmul is the fp32 SIMT replica's output.

Reference: the DMR loop commits slot 0 after a matching vote
(/root/reference/pkg/src/hetrt/executor.py:268-274); its matmul-shaped bodies
are numpy fp32 (workloads.py:25-58 style), i.e. plain fp32 arithmetic.  Here
slot order comes from the mapper's ranking, so "slot 0" would be whichever
variant ranks first (in steady state the faster tcgen05 TF32 one, ~5e-5
relative error).  The matmul workload ranks its variants by fidelity
(workloads.MATMUL_FIDELITY: SIMT FP32 < 3xBF16 < TF32), and the runtime
commits / votes into the best-ranked agreeing replica.  These tests check,
at the benchmark's 4096^2 shape, that the committed bytes ARE the SIMT
kernel's bytes, and bound the committed result's error against binary64.
"""

import numpy as np
import pytest

from oracle import matmul as omatmul
from oracle import vote as ovote

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

import paper_1405_2912_b200 as hf  # noqa: E402
from paper_1405_2912_b200 import kernels  # noqa: E402

N = 4096


@pytest.fixture(scope="module")
def operands():
    a, b = omatmul.make_inputs(N, seed=11)
    ta, tb = torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda()
    simt = torch.empty(N, N, device="cuda")
    kernels.gemm_simt(ta, tb, simt)
    tc3 = torch.empty(N, N, device="cuda")
    # the launch shape TMR uses on one GPU (replicas share it: co-scheduling
    # shapes, no CTA-pair tail split), so its bytes are the runtime's
    kernels.gemm_tc(ta, tb, tc3, mode=hf._lib.HF_GEMM_3XBF16 | hf._lib.HF_GEMM_COSCHEDULE)
    torch.cuda.synchronize()
    return a, b, ta, tb, simt.cpu().numpy(), tc3.cpu().numpy()


def _runtime(kinds, overrides=None):
    cfg = hf.gpu_fleet_config(devices=(0,), kinds=kinds)
    cfg["memory_spaces"].append({"id": "gpu0ckpt", "device": 0})
    for u in cfg["units"]:
        u.update((overrides or {}).get(u["id"], {}))
    rt = hf.Runtime(hf.load_fleet(cfg), hf.RuntimeConfig(checkpoint_space="gpu0ckpt"))
    task = hf.get_workload("matmul").attach(rt, kinds=kinds)
    return rt, task


def _run(rt, task, ta, tb, strategy, tasks=3):
    vt = hf.ValueType.FLOAT32
    reps, outs = [], []
    for _ in range(tasks):       # several tasks: the mapper's slot order changes as profiles fill
        ia = rt.register_device_data(ta.view(-1).view(torch.uint8).clone(), N * N, vt, "r", "gpu0mem")
        ib = rt.register_device_data(tb.view(-1).view(torch.uint8).clone(), N * N, vt, "r", "gpu0mem")
        ic = rt.register_data(bytes(4 * N * N), N * N, vt, "w")
        reps.append(rt.invoke(task, {"A": ia, "B": ib, "C": ic, "n": N}, hf.Strategy(strategy)))
        outs.append(rt.read_array(ic).reshape(N, N))
    return reps, outs


def test_dmr_commits_simt_bytes(operands):
    a, b, ta, tb, simt, _ = operands
    rt, task = _runtime(("gpu-tc", "gpu-simt"))
    reps, outs = _run(rt, task, ta, tb, hf.StrategyKind.HET_DMR)
    for rep, out in zip(reps, outs):
        # whichever slot the mapper's ranking gave the SIMT unit (slot order
        # itself is covered on the CPU: test_runtime_host TestCommitFidelity)
        assert rep.success and rep.votes == ["match"]
        assert rep.committed.kernel == "mm_simt"
        assert out.tobytes() == simt.tobytes()


def test_tmr_tc_fault_corrected_into_simt_bytes(operands):
    a, b, ta, tb, simt, _ = operands
    rt, task = _runtime(("gpu-tc", "gpu-simt", "gpu-tc3"),
                        {"gpu0.tc": {"corrupt_prob": 1.0, "corrupt_mode": "bitflip", "corrupt_bit": 30}})
    reps, outs = _run(rt, task, ta, tb, hf.StrategyKind.HET_TMR, tasks=2)
    for rep, out in zip(reps, outs):
        assert rep.success and rep.votes == ["corrected"]
        assert rep.committed.kernel == "mm_simt"
        assert out.tobytes() == simt.tobytes()


def test_tmr_simt_fault_takes_next_best_value(operands):
    a, b, ta, tb, simt, tc3 = operands
    rt, task = _runtime(("gpu-tc", "gpu-simt", "gpu-tc3"),
                        {"gpu0.simt": {"corrupt_prob": 1.0, "corrupt_mode": "bitflip", "corrupt_bit": 30}})
    reps, outs = _run(rt, task, ta, tb, hf.StrategyKind.HET_TMR, tasks=1)
    rep, out = reps[0], outs[0]
    assert rep.success and rep.votes == ["corrected"]
    (_slot, unit, elem, bit), = rep.injected
    assert unit == "gpu0.simt" and bit == 30
    want = simt.reshape(-1).copy()
    want[elem] = tc3.reshape(-1)[elem]      # 3xBF16 ranks next: its value fills the faulty element
    assert out.reshape(-1).tobytes() == want.tobytes()
    # the reported divergence values are each replica's own: the SIMT entry
    # is the flipped value the kernel read, not the voted value it stored
    # over it in place (hf_vote_result.first_raw0)
    log = rep.rounds_log[0]
    area, idx, vals = log["first_divergence"] if len(log["first_divergence"]) == 3 else (None, None, None)
    assert idx == elem
    flipped = simt.reshape(-1)[elem:elem + 1].copy()
    flipped.view(np.uint32)[0] ^= np.uint32(1 << 30)
    assert vals[log["slots"].index("gpu0.simt")] == float(flipped[0])
    assert vals[log["slots"].index("gpu0.tc3")] == float(tc3.reshape(-1)[elem])


def test_committed_error_vs_binary64(operands):
    """Max relative error of the committed (SIMT) result against the binary64
    product, next to numpy's own fp32 matmul (the reference body's
    arithmetic) on the same operands.  Bound written here: <= 2e-6, and no
    worse than 1.5x numpy fp32 (blocked accumulation: 7.1e-7 vs numpy's
    5.5e-7 at 4096^2; a single 4096-long fp32 chain would be 5.4e-6)."""
    a, b, _ta, _tb, simt, _ = operands
    exact = a.astype(np.float64) @ b.astype(np.float64)
    err_simt = float(np.max(np.abs(simt.astype(np.float64) - exact) / np.abs(exact)))
    err_np = float(np.max(np.abs((a @ b).astype(np.float64) - exact) / np.abs(exact)))
    print(f"max rel err: SIMT {err_simt:.3e}, numpy fp32 {err_np:.3e}")
    assert err_simt <= 2e-6
    assert err_simt <= 1.5 * err_np
    assert ovote.reference_first_divergence(simt.reshape(-1), exact.astype(np.float32).reshape(-1), 1e-3) is None
