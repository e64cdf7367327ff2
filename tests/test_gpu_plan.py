"""BatchPlan: device runs, the chunked host pipeline and CUDA-graph replay
agree with the one-shot batched API (same kernels, same bits)."""
import numpy as np
import pytest
import torch

import paper_2010_00465_b200 as csm
from paper_2010_00465_b200.plan import BatchPlan
from tests._util import cfg2_like, laplacian_wave

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("n,batch", [(64, 96), (100, 40)])
def test_plan_run_and_graph_replay_bitwise(cuda, n, batch):
    rng = np.random.default_rng(700 + n)
    a0 = torch.from_numpy(cfg2_like(rng, batch, n=n)).cuda()
    a1 = torch.from_numpy(cfg2_like(rng, batch, n=n)).cuda()
    plan = BatchPlan(batch, n)
    assert plan.graph_safe
    cos, sin, k, s, st = plan.run(a0)
    ref = csm.cos_sin_batched(a0)
    assert torch.equal(cos, ref.cos_part) and torch.equal(sin, ref.sin_part)
    static = plan.capture(a0)
    static.copy_(a1)  # new data into the graph's static input
    cos, sin, k, s, st = plan.replay()
    torch.cuda.synchronize()
    ref = csm.cos_sin_batched(a1)
    assert torch.equal(cos, ref.cos_part) and torch.equal(sin, ref.sin_part)
    assert torch.equal(k, ref.k) and torch.equal(s, ref.s)


def test_plan_graph_wave(cuda):
    rng = np.random.default_rng(710)
    a, t = laplacian_wave(rng, 8, 48)
    a = torch.from_numpy(a).cuda()
    t = torch.from_numpy(t).cuda()
    plan = BatchPlan(8, 48, wave=True)
    plan.capture(a, t)
    c, s_, k, s, st = plan.replay()
    ref = csm.wave_cos_sin_batched(a, t)
    assert torch.equal(c, ref.cos_part) and torch.equal(s_, ref.sin_part)


def test_plan_tiled_is_not_graph_safe(cuda):
    plan = BatchPlan(4, 200)
    assert not plan.graph_safe
    with pytest.raises(RuntimeError):
        plan.capture(torch.zeros((4, 200, 200), dtype=torch.float64, device="cuda"))


def test_plan_run_host_matches(cuda):
    rng = np.random.default_rng(720)
    a = torch.from_numpy(cfg2_like(rng, 256, n=64)).pin_memory()
    c = torch.empty_like(a).pin_memory()
    s = torch.empty_like(a).pin_memory()
    plan = BatchPlan(256, 64, chunk=64)
    plan.run_host(a, c, s, chunks=4)
    torch.cuda.synchronize()
    ref = csm.cos_sin_batched(a.numpy())
    assert np.array_equal(c.numpy(), ref.cos_part) and np.array_equal(s.numpy(), ref.sin_part)


def test_plan_run_host_back_to_back_calls(cuda):
    """Consecutive run_host calls overlap across the call boundary; each
    call's results still belong to its own input."""
    rng = np.random.default_rng(730)
    a1 = torch.from_numpy(cfg2_like(rng, 512, n=64)).pin_memory()
    a2 = torch.from_numpy(cfg2_like(rng, 512, n=64)).pin_memory()
    c1, s1 = torch.empty_like(a1).pin_memory(), torch.empty_like(a1).pin_memory()
    c2, s2 = torch.empty_like(a1).pin_memory(), torch.empty_like(a1).pin_memory()
    plan = BatchPlan(512, 64)
    for _ in range(3):
        plan.run_host(a1, c1, s1, chunks=16)
        plan.run_host(a2, c2, s2, chunks=16)
    torch.cuda.synchronize()
    r1 = csm.cos_sin_batched(a1.numpy())
    r2 = csm.cos_sin_batched(a2.numpy())
    assert np.array_equal(c1.numpy(), r1.cos_part) and np.array_equal(s1.numpy(), r1.sin_part)
    assert np.array_equal(c2.numpy(), r2.cos_part) and np.array_equal(s2.numpy(), r2.sin_part)


def test_plan_run_host_wave(cuda):
    rng = np.random.default_rng(740)
    a, t = laplacian_wave(rng, 64, 48)
    a_h = torch.from_numpy(a).pin_memory()
    t_h = torch.from_numpy(t).pin_memory()
    c_h, s_h = torch.empty_like(a_h).pin_memory(), torch.empty_like(a_h).pin_memory()
    plan = BatchPlan(64, 48, wave=True, chunk=16)
    plan.run_host(a_h, c_h, s_h, t_h, chunks=4)
    torch.cuda.synchronize()
    ref = csm.wave_cos_sin_batched(a, t)
    assert np.array_equal(c_h.numpy(), ref.cos_part) and np.array_equal(s_h.numpy(), ref.sin_part)


def test_plan_capture_host_round_trip(cuda):
    """capture_host: H2D, the run and D2H in one CUDA graph; replays with new
    data in the pinned input reproduce cos_sin_batched bit for bit."""
    rng = np.random.default_rng(750)
    plan = BatchPlan(3, 64)
    a_h = torch.from_numpy(cfg2_like(rng, 3, n=64)).pin_memory()
    c_h, s_h = torch.empty_like(a_h).pin_memory(), torch.empty_like(a_h).pin_memory()
    plan.capture_host(a_h, c_h, s_h)
    for _ in range(3):
        a_h.copy_(torch.from_numpy(cfg2_like(rng, 3, n=64)))
        plan.replay_host()
        torch.cuda.synchronize()
        r = csm.cos_sin_batched(a_h.numpy())
        assert np.array_equal(c_h.numpy(), r.cos_part) and np.array_equal(s_h.numpy(), r.sin_part)
    with pytest.raises(ValueError):
        plan.capture_host(torch.zeros(3, 64, 64, dtype=torch.float64), c_h, s_h)
