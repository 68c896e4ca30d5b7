"""GPU: the CLI quantize command on the B200 library (build/colorq_b200,
SURVEY.md §8(f) row f1) against the reference's composition of the same
command (tools/colorq.cpp:96-112) run through oracle/_ref: byte-identical
output PPM, palette text, error image and histogram CSV, the same summary
line (except time), and the reference's exit codes."""
import os
import subprocess

import numpy as np
import pytest

from oracle.oracle import Oracle, available
from paper_1011_0093_b200 import api
from paper_1011_0093_b200.configs import gmm_image

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not available("reference"), reason="oracle/_ref not built")]

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CLI = os.path.join(ROOT, "build", "colorq_b200")


@pytest.fixture(scope="module")
def ref():
    return Oracle("reference")


def _fmt_g6(v):
    return "%.6g" % v


def _run(args, timeout=300):
    return subprocess.run([CLI] + args, capture_output=True, text=True, timeout=timeout)


@pytest.mark.parametrize("method,k", [("wsm-c", 16), ("wsm", 32), ("km-c", 8)])
def test_cli_quantize_byte_identical(method, k, ref, tmp_path):
    img = gmm_image(128, 64, 24, 77)  # P = 8192 (power of two: bit-exact centers)
    src = tmp_path / "in.ppm"
    src.write_bytes(ref.write_ppm(img))
    out, pal, err, hist = (tmp_path / n for n in ("out.ppm", "pal.txt", "err.ppm", "hist.csv"))
    r = _run(["quantize", str(src), "-o", str(out), "-m", method, "-k", str(k), "-s", "3", "--palette", str(pal),
              "--error-image", str(err), "--dump-histogram", str(hist)])
    assert r.returncode == 0, r.stderr
    # the reference CLI: MethodParams defaults, Termination::convergent(1e-4) = cap 1000 (kmeans.hpp:34)
    mode = 1 if method.endswith("-c") else 0
    if method.startswith("km"):  # run_km_full, then map_pixels + mse (tools/colorq.cpp:96-102)
        o = ref.run_km_full(img, k, mode=mode, max_iters=10, eps=1e-4, cap=1000, seed=3)
        mapped, _ = ref.map_pixels(img, o["centers"])
        q = dict(centers=o["centers"], iterations=o["iterations"], mapped=mapped, mse=ref.mse(img, mapped))
    else:
        q = ref.quantize(img, k, mode=mode, max_iters=10, eps=1e-4, cap=1000, seed=3)
    assert out.read_bytes() == ref.write_ppm(q["mapped"])
    assert pal.read_text() == ref.palette_text(q["centers"])
    assert err.read_bytes() == ref.write_ppm(ref.error_image(img, q["mapped"]))
    h = ref.build_histogram(img)
    lines = ["r,g,b,count"] + [f"{(kk >> 16) & 255},{(kk >> 8) & 255},{kk & 255},{c}" for kk, c in
                               zip(h.keys.tolist(), h.counts.tolist())]
    assert hist.read_text() == "\n".join(lines) + "\n"
    fields = dict(f.split("=", 1) for f in r.stdout.split())
    assert fields["method"] == method and fields["k"] == str(k) and fields["seed"] == "3"
    assert int(fields["iterations"]) == q["iterations"]
    assert fields["mse"] == _fmt_g6(q["mse"])
    assert fields["psnr"] == _fmt_g6(20 * np.log10(255 / np.sqrt(q["mse"])))


def test_cli_exit_codes(ref, tmp_path):
    img = gmm_image(32, 16, 4, 5)
    good = tmp_path / "g.ppm"
    good.write_bytes(ref.write_ppm(img))
    bad = tmp_path / "b.ppm"
    bad.write_bytes(b"P3 1 1 255\n1 2 3\n")
    few = tmp_path / "few.ppm"
    few.write_bytes(ref.write_ppm(np.zeros((4, 4, 3), np.uint8)))  # N' = 1
    o = str(tmp_path / "o.ppm")
    assert _run(["quantize", str(tmp_path / "missing.ppm"), "-o", o]).returncode == 2
    assert _run(["quantize", str(bad), "-o", o]).returncode == 2
    assert _run(["quantize", str(good), "-o", o, "-m", "nope"]).returncode == 3
    assert _run(["quantize", str(good), "-o", o, "-m", "mc"]).returncode == 3  # not provided on this path
    assert _run(["quantize", str(good), "-o", o, "-k", "0"]).returncode == 4
    assert _run(["quantize", str(few), "-o", o, "-k", "2"]).returncode == 4  # k > N' (kmeans.hpp:55-56)
    assert _run(["quantize", str(good), "-o", o, "-k", "4"]).returncode == 0


def test_error_image_api(ref):
    rng = np.random.default_rng(9)
    a = rng.integers(0, 256, (37, 29, 3), dtype=np.uint8)
    b = np.clip(a.astype(int) + rng.integers(-80, 80, a.shape), 0, 255).astype(np.uint8)
    np.testing.assert_array_equal(api.error_image(a, b), ref.error_image(a, b))
    q = api.quantize(a, 8, api.Termination.convergent(1e-4, 100), seed=1, error=True)
    np.testing.assert_array_equal(q.error, ref.error_image(a, q.mapped))


def _csv(path):
    lines = open(path).read().strip().splitlines()
    return [ln.split(",") for ln in lines]


def test_cli_bench_matches_reference_harness(ref, tmp_path):
    """`colorq_b200 bench` against the reference's
    run_bench on the same config: the runs, summary and ranks CSVs agree in
    every column except the wall-time ones (elapsed_ms, time_mean_ms,
    time_rank, mean_rank)."""
    paths = []
    for i, (w, h) in enumerate([(64, 32), (32, 32)]):  # powers of two: bit-exact centers
        p = tmp_path / f"img{i}.ppm"
        p.write_bytes(ref.write_ppm(gmm_image(w, h, 12, 40 + i)))
        paths.append(str(p))
    # bench.hpp:106-139: key=value (no blanks around '='), list items trimmed
    cfg = (f"# grid\nimages={paths[0]}, {paths[1]}\n"
           "methods=wsm, wsm-c, km(iters=5), fkm(k_prime=4)\n"
           "k_values=4, 8\nruns=2\nbase_seed=7\n")
    ours, theirs = str(tmp_path / "ours"), str(tmp_path / "ref")
    conf = tmp_path / "bench.conf"
    conf.write_text(cfg + f"output={ours}\n")
    r = _run(["bench", "-c", str(conf), "--threads", "2"])
    assert r.returncode == 0, r.stderr
    ref.run_bench(cfg, theirs)
    skip = {"_runs.csv": {"elapsed_ms"}, "_summary.csv": {"time_mean_ms"}, "_ranks.csv": {"time_rank", "mean_rank"}}
    for suffix, drop in skip.items():
        a, b = _csv(ours + suffix), _csv(theirs + suffix)
        assert a[0] == b[0] and len(a) == len(b)
        keep = [j for j, name in enumerate(a[0]) if name not in drop]
        for ra, rb in zip(a[1:], b[1:]):
            assert [ra[j] for j in keep] == [rb[j] for j in keep], (suffix, ra, rb)


def test_cli_scaling_dist_evals(ref, tmp_path):
    img = gmm_image(64, 32, 12, 44)
    src = tmp_path / "s.ppm"
    src.write_bytes(ref.write_ppm(img))
    r = _run(["scaling", str(src), "-m", "wsm-c", "--k-values", "2,4,8,16"])
    assert r.returncode == 0, r.stderr
    rows = [ln.split(",") for ln in r.stdout.strip().splitlines()]
    assert rows[0] == ["k", "elapsed_ms", "dist_evals"]
    for row in rows[1:]:
        k = int(row[0])
        q = ref.quantize(img, k, mode=1, max_iters=10, eps=1e-4, cap=1000, seed=1)
        assert int(row[2]) == q["dist_evals"]
