"""The kernels' alternative forms, selected by environment switches read once
per process, against the default forms: each form runs in its own process
(tests/_variant_run.py) on the same inputs.

* SDDMM dense part: the direct form (sddmm_dense2_kernel, per-entry CSR
  positions) and the staged form (SGTK_SDDMM_DENSE=staged) store the same
  tf32(a) * tf32(dot) from the same TMEM dots: bit-identical.
* AGNN dense part: TMA tile::gather4 loaders (SGTK_AGNN_GATHER=tma) and
  cp.async loaders land the same operand bits: bit-identical.
* AGNN fused rows (SGTK_AGNN_FUSED=1: a panel's sparse edges in the dense
  kernel's CTA) run the serial form's arithmetic (SGTK_AGNN_SERIAL=1):
  bit-identical to it.
* SpMM dense part, TF32: A built in TMEM (SGTK_SPMM_TM=1, spmm_tm_kernel)
  and A scattered into shared memory (default, spmm_panel_kernel) feed the
  same products in the same K order and fold groups: bit-identical.
* A row with more than 2^20 edges does not fit Panels::dpos: the SDDMM falls
  back to the staged form (checked against the CPU oracle)."""
import os
import subprocess
import sys

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
RUN = os.path.join(ROOT, "tests", "_variant_run.py")


def run(tmp_path, name, env_extra, what):
    out = tmp_path / f"{name}.npz"
    env = dict(os.environ)
    for k in ("SGTK_SDDMM_DENSE", "SGTK_AGNN_GATHER", "SGTK_AGNN_FUSED", "SGTK_AGNN_SERIAL", "SGTK_SPMM_TM"):
        env.pop(k, None)
    env.update(env_extra)
    subprocess.run([sys.executable, RUN, what, str(out)], check=True, env=env, cwd=ROOT, timeout=600)
    return dict(np.load(out))


def test_sddmm_direct_equals_staged(tmp_path):
    a = run(tmp_path, "direct", {}, "sddmm")
    b = run(tmp_path, "staged", {"SGTK_SDDMM_DENSE": "staged"}, "sddmm")
    assert a.keys() == b.keys() and len(a) >= 8
    for k in a:
        assert np.array_equal(a[k], b[k]), k


def test_spmm_tmem_a_equals_smem_a(tmp_path):
    a = run(tmp_path, "tm", {"SGTK_SPMM_TM": "1"}, "spmm")
    b = run(tmp_path, "smem", {}, "spmm")
    assert a.keys() == b.keys() and len(a) >= 20
    for k in a:
        assert np.array_equal(a[k], b[k]), k


def test_agnn_tma_gather_equals_cp(tmp_path):
    a = run(tmp_path, "cp", {}, "agnn")
    b = run(tmp_path, "tma", {"SGTK_AGNN_GATHER": "tma"}, "agnn")
    for k in a:
        assert np.array_equal(a[k], b[k]), k


def test_agnn_fused_equals_serial(tmp_path):
    a = run(tmp_path, "serial", {"SGTK_AGNN_SERIAL": "1"}, "agnn")
    b = run(tmp_path, "fused", {"SGTK_AGNN_FUSED": "1"}, "agnn")
    fused = [k for k in a if k in ("tf32_32", "tf32_20")]  # the fused form: TF32, d <= 32
    assert len(fused) == 2
    for k in fused:
        assert np.array_equal(a[k], b[k]), k


def test_sddmm_hub_row_beyond_dpos(tmp_path):
    r = run(tmp_path, "hub", {}, "hub")
    assert r["dpos_row_edges"] > (1 << 20)
    for k in ("fp32", "tf32"):
        got, want = r[k], r[k + "_oracle"]
        err = np.abs(got.astype(np.float64) - want).max() / max(np.abs(want).max(), 1e-30)
        assert err <= (1e-5 if k == "fp32" else 2.0 ** -10), (k, err)
