"""Robustness of the chained launches and the operand checks (-m gpu):

  * carries between CTAs are tagged words in the caller's workspace.  The tags
    must not be satisfiable by whatever the workspace held before: poisoned
    workspaces (random bytes, NaN payloads in the tag range, a previous call's
    carries under a reset header) must give bit-identical results;
  * the epoch lives in device memory, so a forward + backward captured in a
    CUDA graph and replayed with new inputs matches the eager calls bit for bit;
  * gradient outputs at odd element offsets (no 16-byte alignment) are served
    (scalar stores) instead of faulting;
  * Scan2dOp / train_host reject operands that do not match the descriptor.
"""
import ctypes as C

import numpy as np
import pytest
import torch

from oracle_lib import Oracle, rel_error
from scan_cases import batch_to_torch, make_batch, oracle_bwd, oracle_fwd

# cfg2-like geometry: 13 strips per scan over 12-warp backward CTAs, so the
# backward chains strips across CTAs through tagged global words; 1024 columns
# chain the forward across CTAs as well
SHAPES = [(6, 24, 200, 16), (2, 16, 1024, 16), (3, 20, 90, 5)]


@pytest.fixture(scope="module")
def orc():
    return Oracle()


def _inputs(orc, S, H, W, N, seed):
    b = make_batch(orc, S, H, W, N, seed0=seed, dtype="f32")
    return b, batch_to_torch(b, device="cuda")


def _step(op, ins, dy):
    y = op.forward(*ins).clone()
    g = [t.clone() for t in op.backward(*ins, dy)]
    return [y] + g


def _same(a, b, label):
    for k, (u, v) in enumerate(zip(a, b)):
        assert torch.equal(u, v), f"{label}: output {k} differs"


@pytest.mark.gpu
@pytest.mark.parametrize("S,H,W,N", SHAPES)
def test_poisoned_workspace(orc, S, H, W, N):
    from paper_2412_00678_b200.api import Scan2dOp

    b, (ins, dy) = _inputs(orc, S, H, W, N, 4100 + W)
    op = Scan2dOp(S, H, W, N, device="cuda")
    ref = _step(op, ins, dy)
    torch.cuda.synchronize()
    e = rel_error(ref[0].cpu().numpy(), oracle_fwd(orc, b, "f64"))
    assert e <= 1e-4
    saved_f, saved_b = op.wsf.clone(), op.wsb.clone()
    g = torch.Generator(device="cuda").manual_seed(7)
    poisons = {
        "random bytes": lambda ws: ws.copy_(torch.randint(0, 256, ws.shape, dtype=torch.uint8, device="cuda",
                                                          generator=g)),
        "tag-range NaN payloads": lambda ws: ws.view(torch.int32)[: ws.numel() // 4].copy_(
            torch.randint(0x7FC00001, 0x7FFFFFFD, (ws.numel() // 4,), dtype=torch.int32, device="cuda",
                          generator=g)) if ws.numel() >= 4 else None,
        "previous carries, header reset": None,
    }
    for name, fn in poisons.items():
        for ws, saved in ((op.wsf, saved_f), (op.wsb, saved_b)):
            if fn is None:
                ws.copy_(saved)
                ws[:16].zero_()  # header: ticket, epoch, magic -> "fresh"
            else:
                fn(ws)
        got = _step(op, ins, dy)
        torch.cuda.synchronize()
        _same(ref, got, name)


@pytest.mark.gpu
@pytest.mark.parametrize("S,H,W,N", SHAPES[:2])
def test_cuda_graph_replay(orc, S, H, W, N):
    from paper_2412_00678_b200.api import Scan2dOp

    op = Scan2dOp(S, H, W, N, device="cuda")
    op.check = False
    batches = [_inputs(orc, S, H, W, N, 5000 + 97 * k)[1] for k in range(3)]
    eager = []
    for ins, dy in batches:
        eager.append(_step(op, ins, dy))
    torch.cuda.synchronize()
    # static input buffers + capture (after a warm-up call on a side stream,
    # as torch.cuda.graphs recommends)
    s_ins = [t.clone() for t in batches[0][0]]
    s_dy = batches[0][1].clone()
    side = torch.cuda.Stream()
    side.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(side):
        _step(op, s_ins, s_dy)
    torch.cuda.current_stream().wait_stream(side)
    torch.cuda.synchronize()
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph):
        outs = [op.forward(*s_ins)] + list(op.backward(*s_ins, s_dy))
    for rep in range(2):
        for k, (ins, dy) in enumerate(batches):
            for d, src in zip(s_ins, ins):
                d.copy_(src)
            s_dy.copy_(dy)
            graph.replay()
            torch.cuda.synchronize()
            _same(eager[k], [o.clone() for o in outs], f"replay {rep} batch {k}")


@pytest.mark.gpu
@pytest.mark.parametrize("S,H,W,N", [(3, 20, 200, 16), (2, 12, 40, 8), (2, 10, 30, 5), (4, 14, 56, 1)])
def test_misaligned_gradient_outputs(orc, S, H, W, N):
    from paper_2412_00678_b200 import _native as nat
    from paper_2412_00678_b200.api import Scan2dOp

    b, (ins, dy) = _inputs(orc, S, H, W, N, 6100 + N)
    op = Scan2dOp(S, H, W, N, device="cuda")
    ref = _step(op, ins, dy)
    # the same backward into outputs at an odd element offset
    shapes = [(S, H, W), (S, H, W), (S, N), (S, H, W, N), (S, H, W, N), (S,), (S,)]
    outs = []
    for shp in shapes:
        n = int(np.prod(shp))
        outs.append(torch.full((n + 1,), float("nan"), device="cuda")[1:].view(shp))
    x, z, B, C_, A, D, bias = ins
    p = lambda t: C.c_void_p(t.data_ptr())
    rc = nat.lib.scan2d_backward(C.byref(op.desc), p(x), p(z), p(B), p(C_), p(A), p(D), p(bias),
                                 p(op.residual), p(dy), *[p(o) for o in (outs[0], outs[1], outs[2], outs[3],
                                                                          outs[4], outs[5], outs[6])],
                                 p(op.wsb), op.wsb_bytes, C.c_void_p(torch.cuda.current_stream().cuda_stream))
    assert rc == nat.OK, nat.status_string(rc)
    torch.cuda.synchronize()
    ref_g = oracle_bwd(orc, b, "f64")
    for k, name in enumerate(("dx", "dz", "dA", "dB", "dC", "dD", "dbias")):
        e = rel_error(outs[k].cpu().numpy().reshape(-1), np.asarray(ref_g[name]).reshape(-1))
        assert e <= 1e-4, f"{name}: {e:.3e}"
        assert torch.allclose(outs[k], ref[1 + k], rtol=1e-4, atol=1e-4), name


@pytest.mark.gpu
def test_scan2dop_rejects_bad_operands(orc):
    from paper_2412_00678_b200.api import Scan2dOp

    S, H, W, N = 2, 16, 32, 16
    _, (ins, dy) = _inputs(orc, S, H, W, N, 7000)
    op = Scan2dOp(S, H, W, N, device="cuda")
    op.forward(*ins)
    bad = list(ins)
    bad[0] = ins[0].transpose(1, 2).contiguous().transpose(1, 2)  # same shape, not contiguous
    with pytest.raises(ValueError, match="contiguous"):
        op.forward(*bad)
    bad = list(ins)
    bad[2] = ins[2].double()
    with pytest.raises(ValueError, match="dtype"):
        op.forward(*bad)
    bad = list(ins)
    bad[4] = ins[4][:1]
    with pytest.raises(ValueError, match="shape"):
        op.forward(*bad)
    with pytest.raises(ValueError, match="dy"):
        op.backward(*ins, dy[:1])


@pytest.mark.gpu
def test_train_host_rejects_bad_operands(orc):
    from paper_2412_00678_b200.api import train_host

    S, H, W, N = 2, 8, 16, 4
    b = make_batch(orc, S, H, W, N, seed0=7100, dtype="f32")
    host = [torch.from_numpy(np.ascontiguousarray(v)) for v in (b.x, b.z, b.B, b.C, b.A, b.D, b.bias)]
    bad = list(host)
    bad[4] = host[4][:, :2].contiguous()  # A with the wrong state dimension
    with pytest.raises(ValueError, match="A"):
        train_host(*bad)
    bad = list(host)
    bad[0] = host[0].cuda()
    with pytest.raises(ValueError, match="host"):
        train_host(*bad)
    y = train_host(*host)[0]  # synchronised on return
    e = rel_error(y.numpy(), oracle_fwd(orc, b, "f64"))
    assert e <= 1e-4
