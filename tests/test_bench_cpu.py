"""CPU checks of the bench harness (no GPU): the reference arm runs the
unmodified reference on the same inputs as the GPU arm and never loads the
product library; both arms' graph generators are the same code."""
import json
import os
import subprocess
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF_SO = os.path.join(ROOT, "oracle", "_ref", "libsgtk_ref.so")

needs_ref = pytest.mark.skipif(not os.path.exists(REF_SO), reason="make -C oracle ref")


@needs_ref
@pytest.mark.parametrize("n,picks,alpha,p_local", [(5000, 7.0, 2.0, 0.9), (3000, 3.0, 0.0, 0.0),
                                                   (20000, 12.0, 4.0, 0.5)])
def test_reference_generator_matches_product(n, picks, alpha, p_local):
    import paper_2412_12218_b200 as sg
    from oracle.oracle import RefLib

    a = RefLib().synth_graph(n, picks, alpha, p_local, 4.0, 3)
    b = sg.synth_graph(n, picks, alpha, p_local, 4.0, 3)
    assert np.array_equal(a.node_pointer, b.node_pointer)
    assert np.array_equal(a.edge_list, b.edge_list)


@needs_ref
def test_reference_inputs_match_product_streams():
    import paper_2412_12218_b200 as sg
    from oracle.oracle import RefLib

    R = RefLib()
    assert np.array_equal(R.dense_random(50, 7, 8), sg.dense_random(50, 7, 8))
    for (w1, r1), (w2, r2) in zip(R.random_gcn_layers(33, 16, 7, 3, 1),
                                  sg.random_gcn_layers(33, 16, 7, 3, 1)):
        assert np.array_equal(w1, w2) and r1 == r2


@needs_ref
@pytest.mark.parametrize("workload", ["cora-gcn", "pubmed-agnn"])
def test_reference_arm_is_clean(tmp_path, workload):
    csv = tmp_path / "r.csv"
    env = dict(os.environ, SGTK_BENCH_PRINT_MAPS="1")
    p = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference",
                        "--workload", workload, "--steps", "2", "--warmup", "1", "--csv", str(csv)],
                       capture_output=True, text=True, env=env, timeout=300)
    assert p.returncode == 0, p.stderr
    line = json.loads(p.stdout.strip().splitlines()[-1])
    assert line["impl"] == "reference" and line["steps"] == 2 and line["warmup"] == 1
    assert line["cpu_baseline"]["kind"] == "reference" and line["dtype"] == "tf32"
    assert line["e2e"]["h2d_bytes_per_step"] == 0
    assert line["max_rel_err_sampled"] < 2e-3
    loaded = [ln for ln in p.stderr.splitlines() if ln.startswith("[bench] loaded:")][0]
    assert "libsgtk_ref.so" in loaded and "libsgtk_b200.so" not in loaded
    rows = csv.read_text().splitlines()
    assert rows[0].startswith("dataset,kernel,path,median_ms,blocks,capacity,nnz,density,"
                              "max_rel_err,gpus,achieved_GBps")
    assert rows[1].split(",")[8] != ""  # max_rel_err filled
