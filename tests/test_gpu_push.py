"""The single-cluster panel's delivery modes perform the same arithmetic and must
give bit-identical L, tau and pivots:
  * panel_push_kernel, pivot row by one multicast bulk copy (default) vs by the
    speculative st.async push of every candidate row (SKL_PUSH_MCAST=0);
  * panel_cluster_kernel push mode (SKL_PANEL_V2=0) vs its L2 row exchange
    (SKL_PANEL_V2=0 SKL_PANEL_PUSH=0).
Across the two kernels (and across the gemv's threads-per-row split, SKL_PUSH_TPR)
only the summation order of A z differs: pivots identical, L and tau within the
north star's 1e-10 * n.  All runs are held to the oracle by test_gpu_blocked.py /
test_gpu_twostep.py."""
import os
import subprocess
import sys
from pathlib import Path

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parent.parent


def run(tmp_path, tag, **env_extra):
    out = tmp_path / f"{tag}.npz"
    env = dict(os.environ, **{k: str(v) for k, v in env_extra.items()})
    p = subprocess.run([sys.executable, str(ROOT / "tests" / "push_worker.py"), str(out)], cwd=ROOT, env=env,
                       capture_output=True, text=True, timeout=600)
    assert p.returncode == 0 and "PUSH_OK" in p.stdout, p.stdout[-2000:] + p.stderr[-4000:]
    return np.load(out)


def same(a, b):
    assert sorted(a.files) == sorted(b.files)
    for k in a.files:
        assert np.array_equal(a[k], b[k]), k


def close(a, b):
    for k in a.files:
        if k[0] == "p":
            assert np.array_equal(a[k], b[k]), k
        else:
            n = a[k].shape[0]
            assert np.allclose(np.tril(a[k], -1) if a[k].ndim == 2 else a[k],
                               np.tril(b[k], -1) if b[k].ndim == 2 else b[k], rtol=1e-10 * n, atol=1e-10 * n), k


def test_multicast_bit_identical_to_dsmem_push(tmp_path):
    # the DSMEM push reserves 16 row slots in shared memory: pin the GPU panel widths so
    # both runs use the same plan (the factorization is only bit-stable for a fixed plan)
    pin = dict(SKL_GPU_NB=80)
    same(run(tmp_path, "mc", SKL_PUSH_MCAST=1, **pin), run(tmp_path, "dp", SKL_PUSH_MCAST=0, **pin))


def test_old_kernel_push_bit_identical_to_l2_exchange(tmp_path):
    same(run(tmp_path, "o1", SKL_PANEL_V2=0, SKL_PANEL_PUSH=1), run(tmp_path, "o0", SKL_PANEL_V2=0, SKL_PANEL_PUSH=0))


def test_lean_kernel_matches_old_kernel_and_tpr(tmp_path):
    new = run(tmp_path, "new")
    close(new, run(tmp_path, "old", SKL_PANEL_V2=0))
    close(new, run(tmp_path, "tpr1", SKL_PUSH_TPR=1))


def test_small_tile_gemm_bit_identical(tmp_path):
    # trailing updates with few 128x128 tiles run on 64x64-tile CTAs (gemm_lower_small_kernel):
    # same DMMA k order per element, one add into C -> bit-identical factors
    same(run(tmp_path, "small", SKL_GEMM_SMALL_TILES=296), run(tmp_path, "big", SKL_GEMM_SMALL_TILES=0))



def test_fused_epilogue_bit_identical_to_separate_launches(tmp_path):
    # panel_finish_pack_kernel packs P / Q straight from the panel buffer and writes the same
    # W entries as finish_gather + finish_write + pack_rankk: the whole factorization must not
    # change by a bit (SKL_FUSED_FINISH=0 keeps the three launches)
    same(run(tmp_path, "fz", SKL_TEST_BIG=1), run(tmp_path, "f0", SKL_FUSED_FINISH=0, SKL_TEST_BIG=1))


def test_small_tile_gemm_bit_identical_to_large_tiles(tmp_path):
    # the 64x64-tile trailing GEMM accumulates every element in the same k order as the
    # 128x128-tile kernel (the driver switches between them by size)
    same(run(tmp_path, "gs", SKL_GEMM_SMALL_TILES=100000), run(tmp_path, "gl", SKL_GEMM_SMALL_TILES=0))
