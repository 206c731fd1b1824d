"""Pins of the CPU oracle against things other than itself (no GPU needed).

Each test names the passage or closed form it checks.  Together they make a
dropped term, a wrong sign, a transposed operand or a wrong constant in
oracle/oracle.c fail somewhere (DESIGN.md §5 maps outputs -> pins).
"""
import json
import math
import os

import numpy as np
import pytest
from scipy import integrate

import oracle
import synth

GAMMA = synth.GAMMA
PI = math.pi


def _W(r, h):
    return oracle.kernel(r, h, GAMMA)[0]


# --------------------------------------------------------------------------
# Kernel (reading R1): normalisation, second moment, shape, derivatives.
# --------------------------------------------------------------------------
@pytest.mark.parametrize("h", [0.01, 0.077175, 1.0, 3.5])
def test_kernel_integrates_to_one(h):
    """int_0^H 4 pi r^2 W(r,h) dr = 1 (BASELINE north_star: 'the kernel integrates to 1')."""
    H = GAMMA * h
    val, err = integrate.quad(lambda r: 4 * PI * r * r * _W(r, h), 0, H, points=[H / 2], epsabs=0, epsrel=1e-13)
    assert abs(val - 1.0) < 1e-12


def test_kernel_second_moment_sets_gamma():
    """<r^2> = 3 (h/2)^2, i.e. sigma = h/2: the meaning of gamma = 1.825742."""
    h = 0.7
    H = GAMMA * h
    m2, _ = integrate.quad(lambda r: 4 * PI * r ** 4 * _W(r, h), 0, H, points=[H / 2], epsrel=1e-13)
    assert abs(m2 / (3 * (h / 2) ** 2) - 1.0) < 2e-6   # gamma is quoted to 7 digits


def test_kernel_centre_and_half_support():
    """W(0,h) = 0.41842911446446380/h^3 and W(H/2) = W(0)/4."""
    for h in (0.03125, 0.5, 2.0):
        W0 = _W(0.0, h)
        assert abs(W0 * h ** 3 / 0.41842911446446380 - 1) < 1e-14
        WH2 = _W(GAMMA * h / 2, h)
        assert abs(WH2 * h ** 3 / 0.10460727861611595 - 1) < 1e-14
        assert abs(WH2 / W0 - 0.25) < 1e-14


def test_kernel_compact_support_and_continuity():
    """W, dW/dr vanish at and beyond H; both branches agree at x = 1/2."""
    h = 0.3
    H = GAMMA * h
    for r in (H, H * 1.0000001, 2 * H):
        W, dr, dh = oracle.kernel(r, h, GAMMA)
        assert W == 0.0 and dr == 0.0 and dh == 0.0
    eps = 1e-12 * H
    lo = oracle.kernel(H / 2 - eps, h, GAMMA)
    hi = oracle.kernel(H / 2 + eps, h, GAMMA)
    for a, b in zip(lo, hi):
        assert abs(a - b) <= 1e-9 * max(abs(a), 1.0)
    W, dr, dh = oracle.kernel(H * (1 - 1e-6), h, GAMMA)
    assert 0 < W < 1e-15 and dr < 0


@pytest.mark.parametrize("x", [0.05, 0.2, 0.45, 0.55, 0.8, 0.97])
def test_kernel_derivatives_match_finite_differences(x):
    """dW/dr and dW/dh equal central differences of W (pins w' and the h-scaling)."""
    h = 0.4
    r = x * GAMMA * h
    W, dr, dh = oracle.kernel(r, h, GAMMA)
    e = 1e-6 * h
    fd_r = (_W(r + e, h) - _W(r - e, h)) / (2 * e)
    fd_h = (_W(r, h + e) - _W(r, h - e)) / (2 * e)
    assert abs(fd_r - dr) <= 1e-7 * abs(dr) + 1e-9
    assert abs(fd_h - dh) <= 1e-7 * abs(dh) + 1e-9


# --------------------------------------------------------------------------
# Tiny closed-form systems.
# --------------------------------------------------------------------------
def _both(xyzh, vm, nc=3):
    a = oracle.bruteforce(xyzh, vm)
    b = oracle.celllist(xyzh, vm, nc)
    for f in oracle.FIELDS:
        assert np.array_equal(a[f], b[f]), f
    return a


def test_lone_particle():
    """rho = m W(0,h); wcount = W(0,h); h rho_dh/rho = -3; div = curl = 0; nngb = 0."""
    xyzh = np.array([[0.3, 0.6, 0.9, 0.1]], np.float32)
    vm = np.array([[0.4, -1.0, 2.0, 0.25]], np.float32)
    a = _both(xyzh, vm)
    h, m = float(xyzh[0, 3]), float(vm[0, 3])
    W0 = _W(0.0, h)
    assert abs(a["rho"][0] / (m * W0) - 1) < 1e-15
    assert abs(a["wcount"][0] / W0 - 1) < 1e-15
    assert abs(h * a["rho_dh"][0] / a["rho"][0] + 3) < 1e-14
    assert abs(h * a["wcount_dh"][0] / a["wcount"][0] + 3) < 1e-14
    assert a["div_v"][0] == 0 and a["curl_x"][0] == 0 and a["curl_y"][0] == 0 and a["curl_z"][0] == 0
    assert a["nngb"][0] == 0


def test_two_particles_half_support_and_pair_symmetry():
    """At r = H/2 (equal h, m): rho_i = rho_j = m (W(0) + W(0)/4); the rho, wcount,
    rho_dh contributions and rho*div, rho*curl are symmetric."""
    h = 0.125
    H = GAMMA * h
    # put the pair along a skew axis so every component is exercised; r = H/2 in fp64
    d = np.array([3.0, -2.0, 6.0]) / 7.0 * (H / 2)
    p0 = np.array([0.5, 0.5, 0.5])
    xyzh = np.array([[*p0, h], [*(p0 + d), h]], np.float32)
    vm = np.array([[0.3, 0.1, -0.2, 0.5], [-0.1, 0.4, 0.25, 0.5]], np.float32)
    a = _both(xyzh, vm)
    r = float(np.linalg.norm(xyzh[1, :3].astype(np.float64) - xyzh[0, :3].astype(np.float64)))
    assert abs(r / (H / 2) - 1) < 1e-6
    Wr = _W(r, h)
    assert abs(Wr / _W(0, h) - 0.25) < 1e-5
    for f in ("rho", "wcount", "rho_dh", "wcount_dh"):
        assert abs(a[f][0] - a[f][1]) <= 1e-15 * abs(a[f][0])
    assert abs(a["rho"][0] - 0.5 * (_W(0, h) + Wr)) < 1e-13 * a["rho"][0]
    for f in ("div_v", "curl_x", "curl_y", "curl_z"):
        assert abs(a[f][0] * a["rho"][0] - a[f][1] * a["rho"][1]) < 1e-12 * (abs(a[f][0] * a["rho"][0]) + 1e-300)
    assert list(a["nngb"]) == [1, 1]


def test_two_particle_div_curl_closed_form():
    """Two particles: div_i = -m_j (v_ij.x_ij) W'(r)/(r rho_i), curl_i = m_j (v_ij x x_ij) W'(r)/(r rho_i)."""
    h = float(np.float32(0.1))
    xyzh = np.array([[0.40, 0.50, 0.50, h], [0.46, 0.53, 0.48, h]], np.float32)
    vm = np.array([[1.0, 0.0, 0.5, 0.3], [0.0, 2.0, -1.0, 0.7]], np.float32)
    a = _both(xyzh, vm)
    x = xyzh[:, :3].astype(np.float64)
    v = vm[:, :3].astype(np.float64)
    m = vm[:, 3].astype(np.float64)
    xij, vij = x[0] - x[1], v[0] - v[1]
    r = np.linalg.norm(xij)
    W, dWdr, _ = oracle.kernel(r, h, GAMMA)
    rho0 = m[0] * _W(0, h) + m[1] * W
    assert abs(a["rho"][0] / rho0 - 1) < 1e-14
    div = -m[1] * np.dot(vij, xij) * dWdr / r / rho0
    curl = m[1] * np.cross(vij, xij) * dWdr / r / rho0
    assert abs(a["div_v"][0] - div) < 1e-13 * abs(div)
    for k, f in enumerate(("curl_x", "curl_y", "curl_z")):
        assert abs(a[f][0] - curl[k]) < 1e-13 * np.abs(curl).max()


@pytest.mark.parametrize("x", [0.2, 0.45, 0.6, 0.9, 0.995])
def test_condition_scale_matches_radial_finite_difference(x):
    """c_div - a_div = |d(rho div)/d ln r| for one pair (reading R14): the div term of a pair
    scales as w'(r/H) along a fixed direction, so its log-derivative is x w''/w'."""
    h = 0.0625
    H = GAMMA * h
    u = np.array([2.0, -1.0, 2.0]) / 3.0
    p0 = np.array([0.5, 0.5, 0.5])
    v = np.array([[0.25, -0.5, 1.0, 0.5], [-1.0, 0.75, 0.125, 0.25]], np.float32)

    def D(scale):
        xyzh = np.array([[*p0, h], [*(p0 + u * x * H * scale), h]], np.float32)
        a = oracle.bruteforce(xyzh, v)
        d = xyzh[1, :3].astype(np.float64) - xyzh[0, :3].astype(np.float64)
        return a["div_v"][0] * a["rho"][0], a, np.linalg.norm(d)

    eps = 1e-4
    d0, a0, r0 = D(1.0)
    d1, _, r1 = D(1.0 + eps)
    d2, _, r2 = D(1.0 - eps)
    dlog = np.log(r1 / r2)
    sens = abs(d1 - d2) / dlog                       # |d(rho div)/d ln r|
    expect = (a0["c_div"][0] - a0["a_div"][0]) * a0["rho"][0]
    assert abs(sens - expect) <= 2e-3 * expect + 1e-12


# --------------------------------------------------------------------------
# Tolerance scales (readings R13, R14): A = sum_j |term_ij|, C = sum_j |term_ij| kappa_ij.
# Each scale is pinned where a sum of |terms| has a closed form in terms of outputs that
# are pinned themselves (or of W(0,h) = 0.41842911446446380/h^3), so multiplying any of
# them by a constant (or dropping the self term) fails a test here.
# --------------------------------------------------------------------------
W0_COEF = 0.41842911446446380      # W(0,h) h^3 = 8/(pi gamma^3) (mpmath)


def test_scale_rho_dh_lone_particle():
    """Lone particle: the sums hold only the self term -3 m W(0,h)/h, so
    A^rho_dh = 3 m W(0,h)/h and A^wcount_dh = 3 W(0,h)/h exactly; div/curl scales are 0."""
    for h, m in ((0.1, 0.25), (0.0078125, 2.0 ** -20)):
        xyzh = np.array([[0.3, 0.6, 0.9, h]], np.float32)
        vm = np.array([[0.4, -1.0, 2.0, m]], np.float32)
        a = _both(xyzh, vm)
        h32, m32 = float(xyzh[0, 3]), float(vm[0, 3])
        W0 = W0_COEF / h32 ** 3
        assert abs(a["a_rho_dh"][0] / (3 * m32 * W0 / h32) - 1) < 1e-14
        assert abs(a["a_wcount_dh"][0] / (3 * W0 / h32) - 1) < 1e-14
        assert a["a_rho_dh"][0] == -a["rho_dh"][0] and a["a_wcount_dh"][0] == -a["wcount_dh"][0]
        assert a["a_div"][0] == 0 and a["a_curl"][0] == 0 and a["c_div"][0] == 0 and a["c_curl"][0] == 0


@pytest.mark.parametrize("x", [0.3, 0.45, 0.6, 0.85])
def test_scale_rho_dh_pair_signs(x):
    """Two particles: dW/dh of the pair term has the sign of -(3w + x w') = -(18x^3 - 15x^2 + 3/2)
    for x < 1/2 and +3(1-x)^2(2x-1) for x > 1/2, the self term is -3 m_i W(0,h_i)/h_i < 0.
    Same signs (x < 1/2): A = -rho_dh.  Opposite signs (x > 1/2): A = rho_dh + 6 m_i W(0,h_i)/h_i."""
    h = 0.0625
    H = GAMMA * h
    u = np.array([1.0, 2.0, 2.0]) / 3.0
    p0 = np.array([0.5, 0.5, 0.5])
    xyzh = np.array([[*p0, h], [*(p0 + u * x * H), h]], np.float32)
    vm = np.array([[0.0, 0.0, 0.0, 0.375], [0.0, 0.0, 0.0, 0.625]], np.float32)
    a = _both(xyzh, vm)
    h32, mi = float(xyzh[0, 3]), float(vm[0, 3])
    self_rho = 3 * mi * W0_COEF / h32 ** 4
    self_wc = 3 * W0_COEF / h32 ** 4
    assert list(a["nngb"]) == [1, 1]
    if x < 0.5:
        assert abs(a["a_rho_dh"][0] + a["rho_dh"][0]) <= 1e-14 * a["a_rho_dh"][0]
        assert abs(a["a_wcount_dh"][0] + a["wcount_dh"][0]) <= 1e-14 * a["a_wcount_dh"][0]
    else:
        assert abs(a["a_rho_dh"][0] - (a["rho_dh"][0] + 2 * self_rho)) <= 1e-13 * a["a_rho_dh"][0]
        assert abs(a["a_wcount_dh"][0] - (a["wcount_dh"][0] + 2 * self_wc)) <= 1e-13 * a["a_wcount_dh"][0]
        assert a["a_rho_dh"][0] > -a["rho_dh"][0]


def test_scale_div_single_term_and_cancelling_pair():
    """One neighbour: A^div = |div| (a single term).  Two mirror neighbours whose div terms
    cancel exactly: div = 0 and rho A^div = 2 x (rho A^div of the single pair, same term)."""
    h = 0.0625
    H = GAMMA * h
    d = np.array([1 / 64, 3 / 128, -1 / 32])      # dyadic (exact mirror images in fp32), |d| < H
    p0 = np.array([0.5, 0.5, 0.5])
    v0 = np.array([0.5, -0.25, 1.0])
    vj = np.array([-1.0, 0.75, 0.125])
    one = _both(np.array([[*p0, h], [*(p0 + d), h]], np.float32),
                np.array([[*v0, 0.5], [*vj, 0.25]], np.float32))
    assert one["div_v"][0] != 0
    assert abs(one["a_div"][0] - abs(one["div_v"][0])) <= 1e-15 * abs(one["div_v"][0])
    # k at -d with v_k = v_j: (v_i - v_k).(x_i - x_k) = -(v_i - v_j).(x_i - x_j)
    two = _both(np.array([[*p0, h], [*(p0 + d), h], [*(p0 - d), h]], np.float32),
                np.array([[*v0, 0.5], [*vj, 0.25], [*vj, 0.25]], np.float32))
    assert abs(two["div_v"][0]) <= 1e-15 * two["a_div"][0]
    lhs = two["a_div"][0] * two["rho"][0]
    rhs = 2 * one["a_div"][0] * one["rho"][0]
    assert abs(lhs - rhs) <= 1e-14 * rhs


@pytest.mark.parametrize("perp", [True, False])
def test_scale_curl_single_term(perp):
    """One neighbour: A^curl = m_j |v_ij| |x_ij| |W'|/(r rho); the curl vector has norm
    m_j |v_ij x x_ij| |W'|/(r rho), so A^curl sin(theta) = |curl| (theta = angle(v_ij, x_ij))."""
    h = 0.0625
    H = GAMMA * h
    d = np.array([0.25, 0.5, 0.25]) * H
    p0 = np.array([0.5, 0.5, 0.5])
    vij = np.array([1.0, -1.0, 1.0]) if perp else np.array([1.0, 0.25, -0.5])   # (1,-1,1).(1,2,1) = 0
    xyzh = np.array([[*p0, h], [*(p0 + d), h]], np.float32)
    vm = np.array([[*vij, 0.5], [0.0, 0.0, 0.0, 0.25]], np.float32)
    a = _both(xyzh, vm)
    x = xyzh[:, :3].astype(np.float64)
    xij = x[0] - x[1]
    v = vm[0, :3].astype(np.float64)
    sin = np.linalg.norm(np.cross(v, xij)) / (np.linalg.norm(v) * np.linalg.norm(xij))
    cn = np.sqrt(a["curl_x"][0] ** 2 + a["curl_y"][0] ** 2 + a["curl_z"][0] ** 2)
    assert cn > 0
    assert abs(a["a_curl"][0] * sin - cn) <= 1e-13 * cn
    if perp:
        assert abs(sin - 1) < 1e-12


@pytest.mark.parametrize("x", [0.2, 0.6, 0.9, 0.995])
def test_condition_scale_curl_matches_radial_finite_difference(x):
    """c_curl - a_curl = |d(rho curl)/d ln r| for one pair with v_ij perpendicular to x_ij
    (reading R14; the curl analogue of the c_div pin): rho curl = m (v x u) r W'(r)/r
    along a fixed unit direction u, whose log-derivative in r is x w''/w'."""
    h = 0.0625
    H = GAMMA * h
    u = np.array([2.0, 1.0, 2.0]) / 3.0
    p0 = np.array([0.5, 0.5, 0.5])
    v = np.array([[1.0, 0.0, -1.0, 0.5], [0.0, 0.0, 0.0, 0.25]], np.float32)   # (1,0,-1).(2,1,2) = 0

    def R(scale):
        xyzh = np.array([[*p0, h], [*(p0 + u * x * H * scale), h]], np.float32)
        a = oracle.bruteforce(xyzh, v)
        d = xyzh[1, :3].astype(np.float64) - xyzh[0, :3].astype(np.float64)
        c = np.array([a["curl_x"][0], a["curl_y"][0], a["curl_z"][0]]) * a["rho"][0]
        return c, a, np.linalg.norm(d)

    eps = 1e-4
    c0, a0, _ = R(1.0)
    c1, _, r1 = R(1.0 + eps)
    c2, _, r2 = R(1.0 - eps)
    sens = np.linalg.norm(c1 - c2) / np.log(r1 / r2)
    expect = (a0["c_curl"][0] - a0["a_curl"][0]) * a0["rho"][0]
    assert abs(sens - expect) <= 2e-3 * expect + 1e-12
    # and A^curl itself: a single perpendicular term, A = |curl|
    assert abs(a0["a_curl"][0] * a0["rho"][0] - np.linalg.norm(c0)) <= 1e-12 * np.linalg.norm(c0)


def test_asymmetric_cutoffs():
    """H_j < r < H_i: i counts j, j does not count i (gather with h_i)."""
    xyzh = np.array([[0.5, 0.5, 0.5, 0.05], [0.58, 0.5, 0.5, 0.02]], np.float32)
    vm = np.array([[0, 0, 0, 1], [0, 0, 0, 1]], np.float32)
    a = _both(xyzh, vm)
    assert list(a["nngb"]) == [1, 0]


def test_coincident_particles_have_no_gradient_term():
    """r = 0, j != i (reading R7): j counts as a neighbour with W(0), gradient term 0."""
    xyzh = np.array([[0.5, 0.5, 0.5, 0.0625], [0.5, 0.5, 0.5, 0.0625]], np.float32)
    vm = np.array([[1, 0, 0, 1], [0, 1, 0, 1]], np.float32)
    a = _both(xyzh, vm)
    assert list(a["nngb"]) == [1, 1]
    assert abs(a["rho"][0] / (2 * _W(0, 0.0625)) - 1) < 1e-15
    assert a["div_v"][0] == 0 and a["curl_z"][0] == 0


def test_band_pair_is_counted():
    """A pair with |r^2 - H^2| < 1e-6 H^2 is reported in band (BASELINE north_star)."""
    r = 0.0625
    h = np.float32(r / GAMMA)
    xyzh = np.array([[0.5, 0.5, 0.5, h], [0.5 + r, 0.5, 0.5, h]], np.float32)
    vm = np.array([[0, 0, 0, 1], [0, 0, 0, 1]], np.float32)
    a = _both(xyzh, vm)
    assert list(a["band"]) == [1, 1]
    H = GAMMA * float(h)
    assert list(a["nngb"]) == [int(r * r < H * H)] * 2


# --------------------------------------------------------------------------
# Worked example (tests/golden/worked_example_4p.json).
# --------------------------------------------------------------------------
def _load(golden_dir, name):
    with open(os.path.join(golden_dir, name)) as f:
        return json.load(f)


@pytest.mark.parametrize("shift", [0.0, 1.0])
@pytest.mark.parametrize("nc", [3, 8, 16])
def test_worked_example(golden_dir, nc, shift):
    g = _load(golden_dir, "worked_example_4p.json")
    xyzh = np.array(g["xyzh"], np.float32)
    vm = np.array(g["vm"], np.float32)
    if shift:
        xyzh[:, 0] = np.mod(xyzh[:, 0].astype(np.float64) + g["translation_x"], 1.0)
    a = oracle.bruteforce(xyzh, vm)
    b = oracle.celllist(xyzh, vm, nc)
    for f, exp in g["expected"].items():
        exp = np.array(exp, np.float64)
        scale = np.abs(exp).max()
        assert np.all(np.abs(a[f] - exp) <= 1e-13 * np.abs(exp) + 1e-14 * scale), f
        assert np.array_equal(a[f], b[f]), f


# --------------------------------------------------------------------------
# Lattice sums and linear velocity fields (tests/golden/lattice_eta1.2348.json).
# --------------------------------------------------------------------------
def _lattice(side, eta, v_of_x=None, m=None):
    n = side ** 3
    i = np.arange(n)
    ix, iy, iz = i // (side * side), (i // side) % side, i % side
    x = (np.stack([ix, iy, iz], 1) + 0.5) / side
    xyzh = np.zeros((n, 4), np.float32)
    xyzh[:, :3] = x
    xyzh[:, 3] = eta / side
    vm = np.zeros((n, 4), np.float32)
    vm[:, 3] = (1.0 / n) if m is None else m
    if v_of_x is not None:
        vm[:, :3] = v_of_x(xyzh[:, :3].astype(np.float64))
    return xyzh, vm


def test_lattice_density_and_neighbour_count(golden_dir):
    """Uniform lattice: rho = m n (1.0039807835807681), nngb = 56, h rho_dh/rho fixed."""
    g = _load(golden_dir, "lattice_eta1.2348.json")
    side = g["side"]
    xyzh, vm = _lattice(side, g["eta"])
    a = oracle.celllist(xyzh, vm, nc=int(1 / (GAMMA * g["eta"] / side)))
    n = side ** 3
    m = 1.0 / n
    ratio = a["rho"] / (m * n)
    # the golden value is for h = eta/side exactly; the input h is its fp32 rounding, so
    # correct to first order with the (also golden) logarithmic h-derivative
    h32 = float(xyzh[0, 3])
    dlnh = (h32 - g["eta"] / side) / (g["eta"] / side)
    expected = g["rho_over_mn"] * (1 + g["h_rho_dh_over_rho"] * dlnh)
    assert abs(dlnh) < 1e-7
    assert np.all(np.abs(ratio / expected - 1) < g["rel_tol"])
    assert abs(ratio.mean() - 1) < 0.005          # 'a uniform lattice gives rho = m n' (north_star)
    assert np.all(a["nngb"] == g["nngb"])
    h = float(xyzh[0, 3])
    # h rho_dh / rho = -0.0314 is a cancellation of O(3) terms, so the fp32 rounding of h
    # (|dlnh| ~ 1.5e-8) moves it by ~6e-7 relative; 2e-6 still fails any wrong term
    assert np.all(np.abs(h * a["rho_dh"] / a["rho"] / g["h_rho_dh_over_rho"] - 1) < 2e-6)
    t = np.arange(0, n, 97)
    b = oracle.bruteforce(xyzh, vm, targets=t)
    for f in oracle.FIELDS:
        assert np.array_equal(a[f][t], b[f]), f


def test_lattice_linear_velocity(golden_dir):
    """v = A x on the lattice (interior particles): div = S tr(A), curl = S (curl v)_true;
    constant v gives div = curl = 0."""
    g = _load(golden_dir, "lattice_eta1.2348.json")
    side, S = g["side"], g["S_linear_velocity"]
    A = np.array([[0.5, 0.25, -0.125], [0.75, -0.25, 0.375], [0.0625, -0.5, 1.0]])
    xyzh, vm = _lattice(side, g["eta"], lambda x: x @ A.T)
    nc = int(1 / (GAMMA * g["eta"] / side))
    a = oracle.celllist(xyzh, vm, nc)
    H = GAMMA * g["eta"] / side
    x = xyzh[:, :3].astype(np.float64)
    interior = np.all((x > H) & (x < 1 - H), axis=1)
    assert interior.sum() > 1000
    div = a["div_v"][interior]
    assert np.all(np.abs(div / (S * np.trace(A)) - 1) < 1e-6)     # fp32 rounding of v = A x
    curl_true = np.array([A[2, 1] - A[1, 2], A[0, 2] - A[2, 0], A[1, 0] - A[0, 1]])
    for k, f in enumerate(("curl_x", "curl_y", "curl_z")):
        assert np.all(np.abs(a[f][interior] - S * curl_true[k]) < 1e-6 * np.abs(curl_true).max())
    xyzh2, vm2 = _lattice(side, g["eta"], lambda x: np.tile([0.5, -1.25, 2.0], (x.shape[0], 1)))
    c = oracle.celllist(xyzh2, vm2, nc)
    for f in ("div_v", "curl_x", "curl_y", "curl_z"):
        assert np.all(c[f] == 0.0)


# --------------------------------------------------------------------------
# h-derivatives against finite differences of the sums.
# --------------------------------------------------------------------------
def test_h_derivatives_finite_difference():
    """rho_dh and wcount_dh equal central differences of rho, wcount in h_i (gather: only h_i matters)."""
    p = synth.tiny_random_set(11, 300, 4, h_frac=0.9)
    targets = np.arange(0, 300, 7)
    base = oracle.bruteforce(p.xyzh, p.vm, targets=targets)
    for t_idx, i in enumerate(targets):
        h = p.xyzh[i, 3]
        eps = np.float32(h * 2 ** -14)
        vals = []
        for hh in (h + eps, h - eps):
            q = p.xyzh.copy()
            q[i, 3] = hh
            r = oracle.bruteforce(q, p.vm, targets=[i])
            vals.append((r["rho"][0], r["wcount"][0], float(hh)))
        dh = vals[0][2] - vals[1][2]
        fd_rho = (vals[0][0] - vals[1][0]) / dh
        fd_wc = (vals[0][1] - vals[1][1]) / dh
        assert abs(fd_rho - base["rho_dh"][t_idx]) <= 1e-6 * base["a_rho_dh"][t_idx]
        assert abs(fd_wc - base["wcount_dh"][t_idx]) <= 1e-6 * base["a_wcount_dh"][t_idx]


# --------------------------------------------------------------------------
# O1 == O2 and invariances.
# --------------------------------------------------------------------------
def test_bruteforce_equals_celllist_c1():
    p = synth.make("c1")
    a = oracle.bruteforce(p.xyzh, p.vm)
    b = oracle.celllist(p.xyzh, p.vm, p.nc)
    for f in oracle.FIELDS:
        assert np.array_equal(a[f], b[f]), f
    assert 45 < a["nngb"].mean() < 51      # ~48 neighbours (BASELINE configs)


def test_bruteforce_equals_celllist_c2_sample():
    p = synth.make("c2")
    t = np.random.default_rng(5).choice(p.n, 1500, replace=False)
    a = oracle.bruteforce(p.xyzh, p.vm, targets=t)
    b = oracle.celllist(p.xyzh, p.vm, p.nc, targets=t)
    for f in oracle.FIELDS:
        assert np.array_equal(a[f], b[f]), f


@pytest.mark.parametrize("seed", range(6))
def test_bruteforce_equals_celllist_tiny(seed):
    """Random tiny sets incl. particles on cell faces, at x = 0 and x = 1 - 2^-24."""
    nc = 3 + seed % 3
    p = synth.tiny_random_set(seed, 64 + 37 * seed, nc)
    xyzh = p.xyzh.copy()
    Cl = 1.0 / nc
    xyzh[0, 0] = np.float32(Cl)          # exactly on a cell face
    xyzh[1, 1] = 0.0
    xyzh[2, 2] = np.float32(1 - 2 ** -24)
    xyzh[3, :3] = xyzh[4, :3]            # coincident pair
    a = oracle.bruteforce(xyzh, p.vm)
    b = oracle.celllist(xyzh, p.vm, nc)
    for f in oracle.FIELDS:
        assert np.array_equal(a[f], b[f]), f


def test_translation_invariance_bitwise():
    """Translation by (1/2,1/2,1/2) mod 1 is exact on the 2^-24 grid: outputs bitwise identical."""
    p = synth.make("c1")
    q = p.xyzh.copy()
    q[:, :3] = np.mod(q[:, :3].astype(np.float64) + 0.5, 1.0)   # exact on the 2^-24 grid
    a = oracle.celllist(p.xyzh, p.vm, p.nc)
    b = oracle.celllist(q, p.vm, p.nc)
    for f in oracle.FIELDS:
        assert np.array_equal(a[f], b[f]), f


def test_permutation_invariance():
    p = synth.make("c1")
    perm = np.random.default_rng(3).permutation(p.n)
    a = oracle.celllist(p.xyzh, p.vm, p.nc)
    b = oracle.celllist(p.xyzh[perm], p.vm[perm], p.nc)
    for f in ("rho", "wcount", "nngb", "band"):
        assert np.allclose(a[f][perm], b[f], rtol=1e-13, atol=0), f
    for f, s in (("rho_dh", "a_rho_dh"), ("div_v", "a_div"), ("curl_x", "a_curl")):
        assert np.all(np.abs(a[f][perm] - b[f]) <= 1e-13 * a[s][perm]), f


def test_galilean_boost():
    """v += u0 leaves div v and curl v unchanged (v_ij only)."""
    p = synth.make("c1")
    vm2 = p.vm.copy()
    vm2[:, :3] += np.float32([0.5, -0.25, 1.0])
    a = oracle.celllist(p.xyzh, p.vm, p.nc)
    b = oracle.celllist(p.xyzh, vm2, p.nc)
    for f, s in (("div_v", "a_div"), ("curl_x", "a_curl"), ("curl_y", "a_curl"), ("curl_z", "a_curl")):
        assert np.all(np.abs(a[f] - b[f]) <= 1e-6 * a[s]), f
    assert np.array_equal(a["rho"], b["rho"])


# --------------------------------------------------------------------------
# Directions, keys, binning, pseudo-Verlet counts and the paper's statistics.
# --------------------------------------------------------------------------
def test_thirteen_directions():
    """13 symmetry-reduced directions: one of each +/- pair, first nonzero > 0,
    6/2 = 3 face, 12/2 = 6 edge, 8/2 = 4 corner."""
    o = oracle.directions()
    assert o.shape == (13, 3)
    allo = {tuple(v) for v in o} | {tuple(-v) for v in o}
    assert len(allo) == 26 and (0, 0, 0) not in allo
    for v in o:
        first = [c for c in v if c != 0][0]
        assert first > 0
    kinds = np.count_nonzero(o, axis=1)
    assert sorted(np.bincount(kinds)[1:].tolist()) == [3, 4, 6]


def test_cell_keys_projection_examples():
    """Projection examples (SPEC.md l.62-70 analogue): key = local offset . unit axis."""
    nc = 4
    Cl = 0.25
    xyzh = np.array([[0.25 + 0.0625, 0.5 + 0.125, 0.75 + 0.1875, 0.01]], np.float32)
    k = oracle.cell_keys(xyzh, nc)
    o = oracle.directions()
    u = np.array([0.0625, 0.125, 0.1875])
    for d in range(13):
        assert abs(k[d, 0] - u @ o[d] / np.linalg.norm(o[d])) < 1e-15
    assert abs(k[8, 0] - 0.0625) < 1e-15 and tuple(o[8]) == (1, 0, 0)
    del Cl


def test_bin_cells_faces_and_stability():
    nc = 4
    xyzh = np.array([[0.25, 0.0, 0.999999940, 0.01],     # on the x face of cell 1; z = 1 - 2^-24
                     [0.2499999, 0.5, 0.5, 0.01],
                     [0.25, 0.0, 0.999999940, 0.01],
                     [0.0, 0.0, 0.0, 0.01]], np.float32)
    cell, order, start = oracle.bin_cells(xyzh, nc)
    assert cell[0] == (1 * 4 + 0) * 4 + 3 and cell[1] == (0 * 4 + 2) * 4 + 2 and cell[3] == 0
    assert list(order) == [3, 1, 0, 2]                  # stable: 0 before 2 in the same cell
    assert start[-1] == 4


@pytest.mark.parametrize("seed", range(20))
def test_pv_window_safety(seed):
    """No in-range pair lies outside its pseudo-Verlet window (SPEC.md l.116 SAFETY), and
    pV candidates <= naive candidates (SPEC acceptance 4), on seeded random instances."""
    nc = 3 + seed % 3
    p = synth.tiny_random_set(seed + 100, 200 + 13 * seed, nc, h_frac=1.0, h_jitter=0.5)
    c, unsafe = oracle.pv_counts(p.xyzh, nc, delta=0.0)
    assert unsafe == 0
    assert np.all(c[:, :, 1] <= c[:, :, 0]) and np.all(c[:, :, 2] <= c[:, :, 1])
    b = oracle.bruteforce(p.xyzh, p.vm)
    assert np.array_equal(c[:, :, 2].sum(1), b["nngb"].astype(np.int64))


def test_paper_hit_fractions(golden_dir):
    """a cell list inspects pairs of which <= 16 % are in range
    (27-cell block at C_l = h: 4 pi/81); ~68 % of pseudo-Verlet
    candidates are in range (face pairs at C_l = h)."""
    g = _load(golden_dir, "paper_statistics.json")
    nc = 8
    h = np.float32((1.0 / nc) / GAMMA)
    while float(h) * GAMMA > 1.0 / nc:
        h = np.nextafter(h, np.float32(0))
    p = synth.uniform_set("stat", 77, 80 ** 3 // 4, nc, 0.0, 1.0, h_mean=float(h))
    t = np.arange(0, p.n, 23)
    c, unsafe = oracle.pv_counts(p.xyzh, nc, targets=t)
    assert unsafe == 0
    naive_frac = c[:, :, 2].sum() / c[:, :, 0].sum()
    assert naive_frac <= g["cell_list_fraction_max"]
    assert abs(naive_frac - g["cell_list_fraction_geometric"]) < 0.004
    face = c[:, 1, :].sum(0)
    pv_face = face[2] / face[1]
    assert abs(pv_face - g["pv_face_fraction"]) < g["pv_face_fraction_tol"]
    tot = g["table3_scalar_ms"]
    assert abs(8 * tot["corner"] + 12 * tot["edge"] + 6 * tot["face"] - tot["total"]) < 0.005
