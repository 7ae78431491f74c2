"""The command-line front end (tools/spconv_b200_cli.cpp, SURVEY 8(f) row 1:
transform persistence and the CLI's build / convolve on the device path),
checked against the reference's own CLI tests (proj/tests/CMakeLists.txt:
cli_nnz, cli_verify_smoke, cli_bad_subcommand) and against the compiled
reference: `build` writes the reference's file byte for byte, `convolve`
prints the reference's output grid byte for byte."""
import os
import re
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CLI = os.path.join(ROOT, "tools", "_build", "spconv_b200")


def run(*args, cwd=None):
    if not os.path.exists(CLI):
        pytest.fail("tools/_build/spconv_b200 not built (make cli)")
    return subprocess.run([CLI, *map(str, args)], capture_output=True, text=True, timeout=600, cwd=cwd)


def write_table(path):
    from paper_2411_19419_b200.layers import densenet121_layers
    with open(path, "w") as f:
        f.write("name,m,n,k,s,p\n")
        for L in densenet121_layers():
            f.write(f"{L.name},{L.m},{L.n},{L.k},{L.s},{L.p}\n")


# ---------------------------------------------------------------------------
# CPU: host-only subcommands and argument handling
# ---------------------------------------------------------------------------

def test_cli_nnz_reference_regex():
    """cli_nnz: `nnz --m 3 --n 3 --k 3 --s 1 --p 1` matches "3,3,3,1,1,49,81,"."""
    r = run("nnz", "--m", 3, "--n", 3, "--k", 3, "--s", 1, "--p", 1)
    assert r.returncode == 0, r.stderr
    assert re.search(r"3,3,3,1,1,49,81,", r.stdout)
    assert r.stdout.splitlines()[0] == "m,n,k,s,p,bound,dense_count,savings_ratio"
    assert r.stdout.splitlines()[1] == "3,3,3,1,1,49,81,0.39506172839506171"


def test_cli_nnz_layer_table(tmp_path):
    import paper_2411_19419_b200 as sp
    from paper_2411_19419_b200.layers import densenet121_layers
    table = tmp_path / "layers.csv"
    write_table(table)
    out = tmp_path / "nnz.csv"
    r = run("nnz", "--layers", table, "--out", out)
    assert r.returncode == 0, r.stderr
    lines = out.read_text().splitlines()
    assert lines[0] == "name,m,n,k,s,p,bound,dense_count,savings_ratio"
    layers = densenet121_layers()
    assert len(lines) == 1 + len(layers)
    for L, ln in zip(layers, lines[1:]):
        f = ln.split(",")
        spec = sp.ConvSpec(L.m, L.n, L.k, L.s, L.p)
        dense = spec.m_out * spec.n_out * L.k * L.k
        assert f[0] == L.name and int(f[6]) == sp.nnz_bound(spec) and int(f[7]) == dense


@pytest.mark.parametrize("args,code", [
    (["frobnicate"], 2),                         # cli_bad_subcommand (WILL_FAIL)
    ([], 2),
    (["build", "--m", 4, "--n", 4], 2),          # --k and --out required
    (["nnz", "--m", "x", "--n", 3, "--k", 3], 2),
    (["nnz", "--bogus", 1], 2),
    (["bench", "--format", "xml"], 2),
    (["nnz"], 1),                                # the reference's runtime error
    (["nnz", "--m", 3, "--n", 3, "--k", 9], 1),  # ConvSpec: kernel larger than padded input
])
def test_cli_errors(args, code):
    r = run(*args)
    assert r.returncode == code, (r.stdout, r.stderr)
    assert "error:" in r.stderr


# ---------------------------------------------------------------------------
# GPU: build / convolve / verify on the device path
# ---------------------------------------------------------------------------

def _grid_text(a):
    rows = [" ".join("%.17g" % v for v in row) for row in a]
    return f"{a.shape[0]} {a.shape[1]}\n" + "".join(r + "\n" for r in rows)


@pytest.mark.gpu
@pytest.mark.parametrize("spec,layout", [((40, 33, 3, 1, 1), "csr"), ((57, 43, 5, 2, 2), "csc"),
                                         ((20, 9, 4, 3, 2), "csr")])
def test_cli_build_and_convolve_match_reference(ref, tmp_path, spec, layout):
    m, n, k, s, p = spec
    tf = tmp_path / "t.txt"
    r = run("build", "--m", m, "--n", n, "--k", k, "--s", s, "--p", p, "--seed", 7, "--layout", layout,
            "--out", tf)
    assert r.returncode == 0, r.stderr
    kern = ref.random_normal_kernel(k, 7)
    rt = ref.build(*spec, kern, layout=0 if layout == "csr" else 1)
    assert tf.read_bytes() == rt.write_text()
    assert r.stdout.startswith(f"wrote transform (m={m}, n={n}, k={k}, s={s}, p={p}) layout {layout} nnz ")
    # convolve a reference-generated grid
    a = ref.random_normal_grid(m, n, 9).reshape(m, n)
    inp = tmp_path / "a.txt"
    inp.write_text(_grid_text(a))
    out = tmp_path / "y.txt"
    r = run("convolve", "--transform", tf, "--input", inp, "--out", out)
    assert r.returncode == 0, r.stderr
    mo, no = (m + 2 * p - k) // s + 1, (n + 2 * p - k) // s + 1
    want = rt.convolve(a.reshape(1, -1))[0].reshape(mo, no)
    assert out.read_text() == _grid_text(want)
    # stdout form, and a kernel given as a file
    kf = tmp_path / "k.txt"
    kf.write_text(_grid_text(kern.reshape(k, k)))
    tf2 = tmp_path / "t2.txt"
    assert run("build", "--m", m, "--n", n, "--k", k, "--s", s, "--p", p, "--kernel", kf, "--layout", layout,
               "--out", tf2).returncode == 0
    assert tf2.read_bytes() == tf.read_bytes()
    r = run("convolve", "--transform", tf, "--input", inp)
    assert r.returncode == 0 and r.stdout == _grid_text(want)


@pytest.mark.gpu
def test_cli_verify_smoke(ref):
    """cli_verify_smoke: `verify --max-dim 4 --seeds 1` passes; its counts and
    deviations are the reference's."""
    r = run("verify", "--max-dim", 4, "--seeds", 1)
    assert r.returncode == 0, r.stdout + r.stderr
    want = ref.run_verification(4, 1)
    assert r.stdout.splitlines()[0] == (f"verify: {want['specs']} specs, {want['conv_cases']} convolution cases, "
                                        f"{want['clipped_specs']} specs with padding-only placements")
    assert "max |sparse - reference| = 0\n" in r.stdout and "max |CSR - CSC|         = 0\n" in r.stdout
    assert r.stdout.endswith("verify: OK\n")


@pytest.mark.gpu
def test_cli_bench_report(tmp_path):
    table = tmp_path / "layers.csv"
    table.write_text("name,m,n,k,s,p\nc1,56,56,3,1,1\nc2,28,28,1,1,0\n")
    out = tmp_path / "r.md"
    r = run("bench", "--layers", table, "--trials", 5, "--warmup", 2, "--format", "markdown", "--out", out,
            "--quiet")
    assert r.returncode == 0, r.stderr
    text = out.read_text()
    assert "| c1 | CSR-SpMV |" in text and "| TOTAL | im2col |" in text
