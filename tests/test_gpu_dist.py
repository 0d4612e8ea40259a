"""GPU: the block-cyclic multi-GPU driver (config 5 path).

Parity bar: the distributed factorization equals the single-device driver bit
for bit (same panels, same GEMM tiles and k order; only the owner of each
C column differs) and the reference's pivots on the golden fixtures.
* virtual ranks: G allocations on one device mapped block-cyclically into one
  VA range, every rank's column-filtered GEMM (one process);
* two processes on one device (gloo, host barrier): the real fd export /
  import path of the VMM blocks.
"""
import os
import socket
import subprocess
import sys

import numpy as np
import pytest

import oracle
from paper_2411_09859_b200.inputs import skew_lower

pytestmark = pytest.mark.gpu


def pk():
    import paper_2411_09859_b200 as m
    return m


@pytest.mark.parametrize("n,b,nbd,G", [(300, 32, 64, 2), (300, 32, 64, 3), (1000, 128, 128, 2),
                                       (1000, 96, 200, 4), (777, 64, 100, 3), (513, 64, 512, 2)])
def test_virtual_ranks_bit_identical_to_single_device(n, b, nbd, G):
    import torch
    from paper_2411_09859_b200.dist import ltlt_blk_piv_dist
    x = skew_lower(n, 5 * n + G)
    ctx, L, tau, piv = ltlt_blk_piv_dist(x, b=b, nbd=nbd, virtual_ranks=G)
    torch.cuda.synchronize()
    ref = pk().ltlt_blk_piv(pk().SkewMatrixLower(x), b=b, fused="var1")
    assert np.array_equal(piv.cpu().numpy(), ref.p.pivots)
    assert np.array_equal(tau.cpu().numpy(), ref.t.tau)
    assert np.array_equal(np.tril(L.cpu().numpy(), -1), np.tril(ref.l.data, -1))
    o = oracle.ltlt_blk_piv(x, b=b, fused="var1")
    assert np.array_equal(piv.cpu().numpy(), o.pivots)
    ctx.close()


def test_virtual_ranks_config2_golden(golden):
    """Config 2 (n=4096, nb=128) over 4 virtual ranks, nbd=256: reference pivots,
    tau and Pfaffian from the golden fixture."""
    import torch
    from paper_2411_09859_b200.dist import ltlt_blk_piv_dist
    g = golden("cfg2_n4096_b128.npz")
    n = 4096
    x = skew_lower(n, 0)
    ctx, L, tau, piv = ltlt_blk_piv_dist(x, b=128, nbd=256, virtual_ranks=4)
    torch.cuda.synchronize()
    pv, tv = piv.cpu().numpy(), tau.cpu().numpy()
    assert np.array_equal(pv, g["piv"])
    assert np.allclose(tv, g["tau"], rtol=1e-10 * n, atol=1e-10 * n)
    sign, lg = oracle.pfaffian_slog(tv, pv, n)
    assert sign == g["sign"] and abs(lg - g["logpf"]) <= 1e-10 * abs(g["logpf"])
    ctx.close()


def test_owner_filter_partitions_the_update():
    """Each virtual rank's GEMM writes only its own columns: W after the driver
    with G=3 equals the G=1 run (also exercises the straddling-tile epilogue:
    nbd=100 is not a multiple of the 128-column tiles)."""
    import torch
    from paper_2411_09859_b200.dist import DistLTLT
    n = 640
    x = skew_lower(n, 3)
    outs = []
    for G in (1, 3):
        c = DistLTLT(n, 64, "var1", nbd=100, virtual_ranks=G)
        c.load_input(x)
        L, tau, piv = c.factorize()
        torch.cuda.synchronize()
        outs.append((np.tril(L.cpu().numpy(), -1), tau.cpu().numpy(), piv.cpu().numpy(),
                     np.tril(c.w_view().cpu().numpy(), -1)))
        c.close()
    for a, b in zip(outs[0], outs[1]):
        assert np.array_equal(a, b)


def test_two_processes_share_blocks_over_vmm(tmp_path):
    """torch.distributed.run, 2 ranks on cuda:0, gloo + host barrier: the fd
    exported VMM blocks, the remote panel gathers and the per-rank GEMMs."""
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    out = tmp_path / "dist.npz"
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    n, b, nbd = 900, 64, 128
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.join(root, "tests", "dist_worker.py"),
           str(out), str(n), str(b), str(nbd)]
    r = subprocess.run(cmd, cwd=root, capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    got = np.load(out)
    x = skew_lower(n, 11)
    ref = pk().ltlt_blk_piv(pk().SkewMatrixLower(x), b=b, fused="var1")
    assert int(got["world"]) == 2
    assert np.array_equal(got["piv"], ref.p.pivots)
    assert np.array_equal(got["tau"], ref.t.tau)
    assert np.array_equal(np.tril(got["l"], -1), np.tril(ref.l.data, -1))
