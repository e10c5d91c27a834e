"""GPU: the PyTorch-tensor boundary (north star: "Python with PyTorch tensors
calling a thin C-ABI extension").  Engine.read_* / write_* / set_external_accel
accept torch CUDA tensors and move device to device through cs_read_device /
cs_write_device on the tensor's current stream: bit-identical to the host
path (the reference's numpy readbacks, gpu/engine.py:362-378), with zero
host<->device copies (checked with the CUDA activity trace)."""

import numpy as np
import pytest

import paper_2507_11794_b200 as P

pytestmark = pytest.mark.gpu


def _memcpys(prof):
    return [e.name for e in prof.events() if "Memcpy" in e.name and ("DtoH" in e.name or
                                                                      "HtoD" in e.name)]


def _scene():
    sc = P.build_scene(P.ScenarioConfig("hanging", (67, 45), dt=0.004))
    rng = np.random.default_rng(11)
    pos = (sc.mesh.positions + rng.normal(scale=2e-3, size=sc.mesh.positions.shape)).astype(np.float32)
    vel = rng.normal(scale=0.05, size=pos.shape).astype(np.float32)
    return sc, pos, vel


def test_tensor_in_tensor_out_is_bit_identical_with_zero_host_copies():
    import torch
    from torch.profiler import ProfilerActivity, profile

    sc, pos, vel = _scene()
    host = P.Engine(sc.mesh, params=sc.params)
    dev = P.Engine(sc.mesh, params=sc.params)
    tp = torch.from_numpy(pos).cuda()
    tv = torch.from_numpy(vel).cuda()
    n = sc.mesh.num_nodes
    outs = {k: torch.empty((n, 3), dtype=torch.float32, device="cuda")
            for k in ("pos", "vel", "nrm", "prev")}
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        dev.write_positions(tp)
        dev.write_velocities(tv)
        dev.step_frames(7)
        dev.read_positions(out=outs["pos"])
        dev.read_velocities(out=outs["vel"])
        dev.read_normals(out=outs["nrm"])
        dev.read_previous_positions(out=outs["prev"])
        torch.cuda.synchronize()
    assert _memcpys(prof) == [], _memcpys(prof)
    host.write_positions(pos)
    host.write_velocities(vel)
    host.step_frames(7)
    np.testing.assert_array_equal(outs["pos"].cpu().numpy(), host.read_positions())
    np.testing.assert_array_equal(outs["vel"].cpu().numpy(), host.read_velocities())
    np.testing.assert_array_equal(outs["nrm"].cpu().numpy(), host.read_normals())
    np.testing.assert_array_equal(outs["prev"].cpu().numpy(), host.read_previous_positions())


def test_tensor_boundary_on_other_streams_and_set_stream():
    """Writes and reads enqueued on a side stream, frames on a third stream
    after set_stream: event ordering keeps the results equal to the host path."""
    import torch

    sc, pos, vel = _scene()
    host = P.Engine(sc.mesh, params=sc.params)
    host.write_positions(pos)
    host.write_velocities(vel)
    dev = P.Engine(sc.mesh, params=sc.params)
    side, run = torch.cuda.Stream(), torch.cuda.Stream()
    tp = torch.from_numpy(pos).cuda()
    tv = torch.from_numpy(vel).cuda()
    out = torch.empty_like(tp)
    torch.cuda.synchronize()
    with torch.cuda.stream(side):
        dev.write_positions(tp)
        dev.write_velocities(tv)
    dev.set_stream(run)
    for _ in range(3):
        dev.step_frames(4)
        host.step_frames(4)
        with torch.cuda.stream(side):
            dev.read_positions(out=out)
            got = out.cpu().numpy()  # .cpu() synchronises `side` only
        np.testing.assert_array_equal(got, host.read_positions())


def test_float64_and_collision_buffers_through_tensors():
    import torch

    sc = P.build_scene(P.ScenarioConfig("drop", (24, 24), obstacle="icosphere:2"))
    a = P.Engine(sc.mesh, sc.obstacle, sc.params, pair_budget=10**12, precision="fp64")
    b = P.Engine(sc.mesh, sc.obstacle, sc.params, pair_budget=10**12, precision="fp64")
    rng = np.random.default_rng(2)
    p64 = sc.mesh.positions + rng.normal(scale=1e-3, size=sc.mesh.positions.shape)
    a.write_state64(pos=torch.from_numpy(p64).cuda())
    b.write_state64(pos=p64)
    a.step_frames(80)
    b.step_frames(80)
    out = torch.empty((sc.mesh.num_nodes, 3), dtype=torch.float64, device="cuda")
    np.testing.assert_array_equal(a.read_positions64(out=out).cpu().numpy(), b.read_positions64())
    out32 = torch.empty((sc.mesh.num_nodes, 3), dtype=torch.float32, device="cuda")
    np.testing.assert_array_equal(a.read_velocities(out=out32).cpu().numpy(), b.read_velocities())
    # the fast engine's accumulator / counts between detect and respond
    from paper_2507_11794_b200 import _native as N

    f = P.Engine(sc.mesh, sc.obstacle, sc.params, pair_budget=10**12)
    f.step_frames(150)
    N.check(f._lib.cs_run_pass(f._handle, N.PASS_FORCE_INTEGRATE))
    N.check(f._lib.cs_run_pass(f._handle, N.PASS_DETECT))
    acc = torch.empty((sc.mesh.num_nodes, 3), dtype=torch.int32, device="cuda")
    cnt = torch.empty((sc.mesh.num_nodes,), dtype=torch.int32, device="cuda")
    f.read_accumulator_raw(out=acc)
    f.read_counts(out=cnt)
    np.testing.assert_array_equal(acc.cpu().numpy(), f.read_accumulator_raw())
    np.testing.assert_array_equal(cnt.cpu().numpy(), f.read_counts())
    assert cnt.sum().item() > 0


def test_external_accel_from_a_tensor_and_shape_checks():
    import torch

    from paper_2507_11794_b200 import SimParams, generate_cloth_grid

    eng = P.Engine(generate_cloth_grid(2, 2), params=SimParams(dt=0.5, gravity=(0, 0, 0)))
    eng.set_external_accel(torch.tensor([[4.0, 0.0, 0.0]] * 4, device="cuda"))
    eng.step()
    np.testing.assert_allclose(eng.read_velocities()[:, 0], np.float32(2.0))
    with pytest.raises(ValueError):
        eng.read_positions(out=torch.empty((4, 3), dtype=torch.float64, device="cuda"))
    with pytest.raises(ValueError):
        eng.write_positions(torch.empty((5, 3), dtype=torch.float32, device="cuda"))
