"""scan2d_train_host (host operands, chunked copy/compute pipeline) against the
device-resident path and the oracle (-m gpu)."""
import numpy as np
import pytest
import torch

from oracle_lib import Oracle, rel_error
from scan_cases import batch_to_torch, make_batch, oracle_bwd, oracle_fwd


@pytest.mark.gpu
@pytest.mark.parametrize("shape,chunks", [((10, 24, 40, 16), 3), ((9, 14, 14, 1), 4), ((5, 20, 32, 8), 1),
                                         ((40, 12, 24, 16), 3), ((33, 8, 16, 16), 2)])  # last two: ramped ends
def test_train_host_matches_device_path(shape, chunks):
    from paper_2412_00678_b200.api import Scan2dOp, train_host

    S, H, W, N = shape
    orc = Oracle()
    b = make_batch(orc, S, H, W, N, seed0=900, dtype="f32")
    (x, z, B, C, A, D, bias), dy = batch_to_torch(b, device="cuda")
    op = Scan2dOp(S, H, W, N, device="cuda")
    y = op.forward(x, z, B, C, A, D, bias).clone()
    grads = [t.clone() for t in op.backward(x, z, B, C, A, D, bias, dy)]
    host = [t.cpu().pin_memory() for t in (x, z, B, C, A, D, bias)]
    outs = train_host(*host, dy=dy.cpu().pin_memory(), chunks=chunks)
    torch.cuda.synchronize()
    assert torch.equal(outs[0], y.cpu())
    for got, ref in zip(outs[1:], grads):
        assert torch.equal(got, ref.cpu())
    # and against the fp64 oracle (north_star tolerance)
    assert rel_error(outs[0].numpy(), oracle_fwd(orc, b, "f64")) < 1e-4
    ref = oracle_bwd(orc, b, "f64")
    names = ["dx", "dz", "dA", "dB", "dC", "dD", "dbias"]
    for k, got in zip(names, outs[1:]):
        assert rel_error(got.numpy().reshape(-1), np.asarray(ref[k]).reshape(-1)) < 1e-4, k


@pytest.mark.gpu
def test_train_host_forward_only_and_errors():
    from paper_2412_00678_b200 import _native as nat
    from paper_2412_00678_b200.api import train_host

    orc = Oracle()
    b = make_batch(orc, 4, 16, 16, 4, seed0=3, dtype="f32")
    (x, z, B, C, A, D, bias), _ = batch_to_torch(b, device="cpu")
    outs = train_host(x, z, B, C, A, D, bias, dy=None, chunks=2)
    torch.cuda.synchronize()
    assert outs[1] is None
    assert rel_error(outs[0].numpy(), oracle_fwd(orc, b, "f64")) < 1e-4
    # an invalid descriptor is refused
    import ctypes as ct

    desc = nat.make_desc(4, 16, 16, 4, params_period=3)
    ptrs = [ct.c_void_p(t.data_ptr()) for t in (x, z, B, C, A, D, bias)]
    y = torch.empty_like(x)
    rc = nat.lib.scan2d_train_host(ct.byref(desc), *ptrs, None, ct.c_void_p(y.data_ptr()), *([None] * 7), 2,
                                   None)
    assert rc == nat.EINVAL


@pytest.mark.gpu
@pytest.mark.parametrize("S,H,W,N,P,G,chunks,red", [(12, 20, 40, 16, 4, 4, 3, False), (24, 14, 14, 1, 6, 3, 4, False),
                                                   (16, 16, 24, 8, 16, 4, 2, True), (8, 20, 30, 16, 8, 8, 4, True),
                                                   (36, 10, 20, 4, 3, 2, 0, False)])
def test_train_host_model_layout(S, H, W, N, P, G, chunks, red):
    """Shared B/C and shared parameters through the host path: chunks cut at
    lcm(G, P) scans, the parameter gradients summed over the chunks; against
    the device-resident operator and the fp64 oracle."""
    from paper_2412_00678_b200.api import Scan2dOp, train_host

    orc = Oracle()
    b = make_batch(orc, S, H, W, N, seed0=950, dtype="f32", P=P, G=G)
    (x, z, B, C, A, D, bias), dy = batch_to_torch(b, device="cuda")
    op = Scan2dOp(S, H, W, N, params_period=P, bc_group=G, device="cuda", group_red=red)
    y = op.forward(x, z, B, C, A, D, bias).clone()
    grads = [t.clone() for t in op.backward(x, z, B, C, A, D, bias, dy)]
    host = [t.cpu().pin_memory() for t in (x, z, B, C, A, D, bias)]
    outs = train_host(*host, dy=dy.cpu().pin_memory(), chunks=chunks, group_red=red)
    assert torch.equal(outs[0], y.cpu())
    names = ["dx", "dz", "dA", "dB", "dC", "dD", "dbias"]
    for k, got, dev_ref in zip(names, outs[1:], grads):
        if k in ("dx", "dz") or (k in ("dB", "dC") and not red):
            assert torch.equal(got, dev_ref.cpu()), k  # per-scan / per-group outputs: the same bits
        else:  # sums whose order differs (over chunks; in-kernel reductions)
            assert rel_error(got.numpy().reshape(-1), dev_ref.cpu().numpy().reshape(-1)) < 1e-6, k
    assert rel_error(outs[0].numpy(), oracle_fwd(orc, b, "f64")) < 1e-4
    ref = oracle_bwd(orc, b, "f64")
    for k, got in zip(names, outs[1:]):
        assert rel_error(got.numpy().reshape(-1), np.asarray(ref[k]).reshape(-1)) < 1e-4, k
