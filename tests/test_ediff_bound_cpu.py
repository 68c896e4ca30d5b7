"""CPU check of the error bound behind the large-path scan's difference form
(paper_1011_0093_b200/csrc/wsm.cuh scan_f32e; DESIGN.md §3 "Difference form").

The kernel evaluates diff = fma(a0, m0, fma(a1, m1, fma(a2, m2, w))) for
Delta = D(x, c_t) - D(x, c_p) and certifies its argmin only when the two
smallest differences are more than 4.4e-6 prev + 2.5e-6 apart, on the claim
|diff - Delta| <= E = 36 u prev + 1e-8 = 2.15e-6 prev + 1e-8 for every evaluated entry
(D(c_p, c_t) < 4 prev). Here the arithmetic is emulated in numpy float32 (an
FMA = one float32 rounding of the product-sum taken in float64, exact to far
below the bound) on random and on adversarial inputs: the reflected center
c_t = c_p + 2 (x - c_p), where every magnitude in the bound is at its maximum
(the reference's midpoint case, kmeans.hpp:220-231).
"""
import numpy as np

f32 = np.float32
E_A, E_B = 2.15e-6, 1e-8          # the claimed bound (36 u prev: (4 |w*| + 5 S) u with |w*|, S <= 4 prev)
CERT_A, CERT_B = 4.4e-6, 2.5e-6   # wsm.cuh F32_E_A / F32_E_B: the certificate's margin (> 2 E)


def _worst_ratio(cp, ct, x):
    cf = cp.astype(f32)                                   # c4[p]
    a = (x.astype(f32) - cf).astype(f32)                  # the FP32 differences of the own-center distance
    a64 = a.astype(np.float64)
    prev = (a64[:, 0] * a64[:, 0]).astype(f32).astype(np.float64)
    prev = (a64[:, 1] * a64[:, 1] + prev).astype(f32).astype(np.float64)
    prev = (a64[:, 2] * a64[:, 2] + prev).astype(f32).astype(np.float64)
    keep = (((cp - ct) ** 2).sum(1) < 4 * prev) & (prev > 0)   # evaluated entries only
    g = ct - cf.astype(np.float64)
    h = cp - cf.astype(np.float64)
    w = ((g ** 2).sum(1) - (h ** 2).sum(1)).astype(f32).astype(np.float64)   # ediff_entry
    m = (-2.0 * (ct - cp)).astype(f32).astype(np.float64)
    d = (a64[:, 2] * m[:, 2] + w).astype(f32).astype(np.float64)
    d = (a64[:, 1] * m[:, 1] + d).astype(f32).astype(np.float64)
    d = (a64[:, 0] * m[:, 0] + d).astype(f32).astype(np.float64)
    delta = ((x - ct) ** 2).sum(1) - ((x - cp) ** 2).sum(1)   # FP64: exact to ~1e-10
    err = np.abs(d - delta)[keep]
    bound = (E_A * prev + E_B)[keep]
    assert keep.any()
    return float((err / bound).max())


def test_bound_on_random_neighbours():
    rng = np.random.default_rng(7)
    worst = 0.0
    for _ in range(8):
        n = 250_000
        cp = rng.uniform(0, 255, (n, 3))
        ct = np.clip(cp + rng.normal(0, 30, (n, 3)), 0, 255)
        x = np.clip(np.rint(cp + rng.normal(0, 18, (n, 3))), 0, 255)
        worst = max(worst, _worst_ratio(cp, ct, x))
    assert worst <= 0.75, worst


def test_bound_on_reflected_centers():
    """c_t just inside the break bound, along x - c_p: |w*| and |a.m| both ~4 prev."""
    rng = np.random.default_rng(11)
    worst = 0.0
    for scale in (0.5, 0.9, 0.99, 0.9999):
        n = 250_000
        cp = rng.uniform(60, 195, (n, 3))
        x = np.clip(np.rint(cp + rng.normal(0, 20, (n, 3))), 0, 255)
        ct = cp + 2.0 * scale * (x - cp) + rng.normal(0, 1e-3, (n, 3))
        ok = np.all((ct >= 0) & (ct <= 255), axis=1)
        worst = max(worst, _worst_ratio(cp[ok], ct[ok], x[ok]))
    assert worst <= 1.0, worst


def test_certificate_margin_covers_two_bounds():
    prev = np.array([0.0, 1e-3, 1.0, 500.0, 195075.0])
    assert np.all(CERT_A * prev + CERT_B > 2.0 * (E_A * prev + E_B) * (1 + 2.0 ** -20))
