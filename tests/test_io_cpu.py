"""CPU: the drop-in's host file formats (include/colorq_b200/io.hpp, SURVEY.md
§8(f) row f1) against the reference's own codecs (ppm.hpp:89-149,
palette.hpp:37-74) compiled in oracle/_ref. Driven through build/io_test."""
import os
import subprocess

import numpy as np
import pytest

from oracle.oracle import Oracle, available

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
IO_TEST = os.path.join(ROOT, "build", "io_test")

pytestmark = pytest.mark.skipif(not (available("reference") and os.path.exists(IO_TEST)),
                                reason="oracle/_ref or build/io_test not built")


@pytest.fixture(scope="module")
def ref():
    return Oracle("reference")


def _io(mode, data, tmp_path, name="in"):
    src = tmp_path / f"{name}.bin"
    dst = tmp_path / f"{name}.out"
    src.write_bytes(data)
    r = subprocess.run([IO_TEST, mode, str(src), str(dst)], capture_output=True, text=True, timeout=60)
    assert r.returncode == 0, r.stderr
    out = dst.read_bytes() if dst.exists() else None
    return r.stdout.strip(), out


@pytest.mark.parametrize("w,h", [(1, 1), (7, 3), (64, 33)])
def test_ppm_roundtrip_is_byte_identical(w, h, ref, tmp_path):
    img = np.random.default_rng(w * 100 + h).integers(0, 256, (h, w, 3), dtype=np.uint8)
    data = ref.write_ppm(img)
    status, out = _io("ppm", data, tmp_path)
    assert status == f"ok {w} {h}"
    assert out == data


def test_ppm_header_variants(ref, tmp_path):
    px = bytes(range(12))
    cases = [
        b"P6 2 2 255\n" + px,
        b"P6\n# comment\n2 2\n# another\n255\n" + px,
        b"P6\t2\r2\f255 " + px,
        b"P6 +2 002 255\n" + px + b"trailing",
    ]
    for i, data in enumerate(cases):
        kind, img = ref.read_ppm(data)
        status, out = _io("ppm", data, tmp_path, f"v{i}")
        assert kind == "ok" and status == "ok 2 2"
        assert out == ref.write_ppm(img)


@pytest.mark.parametrize("data", [
    b"", b"   ", b"P3 1 1 255\n\0\0\0", b"P5 1 1 255\n\0", b"P6", b"P6 0 1 255\n", b"P6 1 -1 255\n",
    b"P6 x 1 255\n", b"P6 1 1 65535\n\0\0\0\0\0\0", b"P6 1 1 255", b"P6 2 2 255\n\0\0\0", b"P6 1 1 1x\n",
    b"P6 99999999999 1 255\n", b"P6 1 1 255#\n\0\0\0",
])
def test_ppm_errors_match_reference_kinds(data, ref, tmp_path):
    kind, _ = ref.read_ppm(data)
    status, _ = _io("ppm", data, tmp_path)
    assert status.split()[0] == "err" and kind != "ok"
    assert status.split()[1] == kind


def test_palette_text_roundtrip(ref, tmp_path):
    rng = np.random.default_rng(5)
    C = np.concatenate([rng.uniform(0, 255, (20, 3)), [[0.5, 127.5, 255.0], [1e-12, 3.25, 99.999999999]]])
    text = ref.palette_text(C)
    status, out = _io("palette", text.encode(), tmp_path)
    assert status == f"ok {len(C)}"
    assert out.decode() == text


def test_palette_malformed(tmp_path):
    status, _ = _io("palette", b"1 2 3\n4 5\n", tmp_path)
    assert status.startswith("err runtime malformed palette line")
