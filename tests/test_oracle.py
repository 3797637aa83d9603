"""The CPU oracle (oracle/lbm_oracle.c) pinned before it is trusted:

1. against the reference's own known answers, restated from its unit tests
   (proj/tests/test_descriptor.cpp, test_collision.cpp, test_boundaries.cpp,
   test_reference_lattice.cpp), and
2. against the UNMODIFIED reference solver: committed golden hashes of its
   outputs (tests/golden/golden.json, made by tests/golden/make_golden.py) and,
   where oracle/_ref is built, a bit-for-bit comparison on the same inputs.
"""
import math

import numpy as np
import pytest

from golden_cases import CASES, make_case
from pyoracle import BB, BGK, MBB, NODYN, RR, TRT, Case, Recipe, canonical_hash, descriptor

C19, W19, OPP19 = descriptor(19)
C27, W27, OPP27 = descriptor(27)


def near(a, b, eps):
    """doctest::Approx(b).epsilon(eps) semantics: |a-b| < eps * (1 + max(|a|, |b|))."""
    a, b = np.asarray(a, float), np.asarray(b, float)
    return bool(np.all(np.abs(a - b) < eps * (1.0 + np.maximum(np.abs(a), np.abs(b)))))


def moments(f, q=19):
    c = C19 if q == 19 else C27
    drho = f.sum()
    rho = 1.0 + drho
    j = c.T.astype(float) @ f
    return np.concatenate([[rho], j / rho])


def pi_neq(oracle, f, q=19):
    c = C19 if q == 19 else C27
    m = moments(f, q)
    feq = oracle.equilibrium(q, 2, m[0], m[1:])
    fn = f - feq
    return np.array([np.sum(c[:, a] * c[:, b] * fn) for a, b in ((0, 0), (0, 1), (0, 2), (1, 1), (1, 2), (2, 2))])


def near_eq(oracle, rng, rho, u, noise, q=19):
    return oracle.equilibrium(q, 2, rho, u) + rng.uniform(-noise, noise, q)


# --------------------------------------------------------------- descriptor
@pytest.mark.parametrize("q", [19, 27])
def test_isotropy_and_opposites(q):  # test_descriptor.cpp:66-105
    c, w, opp = descriptor(q)
    assert abs(w.sum() - 1.0) < 1e-15
    assert np.all(np.abs(w @ c) < 1e-16)
    second = np.einsum("i,ia,ib->ab", w, c, c)
    assert np.allclose(second, np.eye(3) / 3.0, atol=1e-15)
    fourth = np.einsum("i,ia,ib,ic,id->abcd", w, c, c, c, c)
    cs4 = 1.0 / 9.0
    d = np.eye(3)
    iso = cs4 * (np.einsum("ab,cd->abcd", d, d) + np.einsum("ac,bd->abcd", d, d) + np.einsum("ad,bc->abcd", d, d))
    assert np.allclose(fourth, iso, atol=1e-15)
    for i in range(q):
        assert opp[opp[i]] == i
        assert np.array_equal(c[opp[i]], -c[i])
    assert np.array_equal(C27[:19], C19)  # D3Q27 extends the frozen D3Q19 order


def test_equilibrium2_known_values(oracle):  # test_descriptor.cpp:106-123
    assert np.all(oracle.equilibrium(19, 2, 1.0, [0, 0, 0]) == 0.0)
    feq = oracle.equilibrium(19, 2, 1.0, [0.1, 0.0, 0.0])
    assert near(feq[0], -0.005, 1e-14)
    assert near(feq[1], -0.015, 1e-14)
    assert near(feq[2], 0.33 / 18.0, 1e-14)
    cs2 = 1.0 / 3.0
    u = np.array([0.1, 0, 0])
    for i in range(19):
        cu = C19[i] @ u
        ref = W19[i] * (1 + cu / cs2 + cu * cu / (2 * cs2 * cs2) - u @ u / (2 * cs2)) - W19[i]
        assert near(feq[i], ref, 1e-14)


@pytest.mark.parametrize("q", [19, 27])
def test_equilibrium4_hermite_series(oracle, q):  # test_descriptor.cpp:140-163
    c, w, _ = descriptor(q)
    cs2 = 1.0 / 3.0
    u = np.array([0.05, 0.02, 0.0])
    feq = oracle.equilibrium(q, 4, 1.0, u)
    for i in range(q):
        ci = c[i].astype(float)
        s = 1.0 + ci @ u / cs2
        for a in range(3):
            for b in range(3):
                s += (ci[a] * ci[b] - (cs2 if a == b else 0.0)) * u[a] * u[b] / (2 * cs2 * cs2)
        for a in range(3):
            for b in range(3):
                for g in range(3):
                    # the reference keeps only the six aab terms (descriptor.hpp:94-97)
                    if len({a, b, g}) != 2:
                        continue
                    h3 = ci[a] * ci[b] * ci[g] - cs2 * (ci[a] * (b == g) + ci[b] * (a == g) + ci[g] * (a == b))
                    s += h3 * u[a] * u[b] * u[g] / (6 * cs2 ** 3)
        assert near(feq[i], w[i] * s - w[i], 1e-13)
    f2 = oracle.equilibrium(q, 4, 1.02, [0.03, -0.04, 0.05])
    m = moments(f2, q)
    assert near(m[0], 1.02, 1e-14) and near(m[1:], [0.03, -0.04, 0.05], 1e-12)


# --------------------------------------------------------------- collisions
def apply(oracle, recipe, f, q=19, dtype=np.float64):
    return oracle.apply(q, recipe, np.asarray(f, dtype)[None, :])[0]


@pytest.mark.parametrize("q", [19, 27])
def test_bgk_known_answers(oracle, q):  # test_collision.cpp:42-80
    rng = np.random.default_rng(5)
    for om in (0.6, 1.0, 1.7):
        fe = oracle.equilibrium(q, 2, 1.01, [0.03, -0.02, 0.01])
        assert near(apply(oracle, Recipe(base=BGK, omega=om), fe, q), fe, 1e-13)
    f0 = near_eq(oracle, rng, 1.0, [0.05, 0.0, -0.01], 1e-2, q)
    m = moments(f0, q)
    rho, u = m[0], m[1:]
    feq = oracle.equilibrium(q, 2, rho, u)
    f = apply(oracle, Recipe(base=BGK, omega=1.7), f0, q)
    assert near(f, f0 - 1.7 * (f0 - feq), 1e-13)
    assert near(moments(f, q), moments(f0, q), 1e-13)


@pytest.mark.parametrize("q", [19, 27])
def test_trt_parity_split(oracle, q):  # test_collision.cpp:82-125
    c, w, opp = descriptor(q)
    rng = np.random.default_rng(13)
    om, lam = 1.2, 3.0 / 16.0
    omm = oracle.derive_omega_minus(om, lam)
    assert near((1 / om - 0.5) * (1 / omm - 0.5), lam, 1e-14)
    f0 = near_eq(oracle, rng, 1.02, [0.03, 0.01, -0.02], 2e-2, q)
    m = moments(f0, q)
    rho, u = m[0], m[1:]
    feq = oracle.equilibrium(q, 2, rho, u)
    f = apply(oracle, Recipe(base=TRT, omega=om, lambda_=lam), f0, q)
    j = opp
    expect = f0 - om * 0.5 * ((f0 + f0[j]) - (feq + feq[j])) - omm * 0.5 * ((f0 - f0[j]) - (feq - feq[j]))
    assert near(f, expect, 1e-12)
    # omega_minus == omega collapses to BGK: lambda = (1/om - 1/2)^2
    lam_b = (1 / 1.4 - 0.5) ** 2
    f1 = near_eq(oracle, rng, 1.0, [0.01, -0.02, 0.04], 1e-2, q)
    assert near(apply(oracle, Recipe(base=TRT, omega=1.4, lambda_=lam_b), f1, q),
                apply(oracle, Recipe(base=BGK, omega=1.4), f1, q), 1e-12)


@pytest.mark.parametrize("q", [19, 27])
def test_rr_known_answers(oracle, q):  # test_collision.cpp:127-180
    rng = np.random.default_rng(17)
    fe4 = oracle.equilibrium(q, 4, 1.01, [0.04, -0.03, 0.02])
    assert near(apply(oracle, Recipe(base=RR, omega=1.6, omega_bulk_ho=1.0), fe4, q), fe4, 5e-13)
    # omega = omega_bulk_ho = 0 isolates the projection: idempotent, reproduces Pi
    # (recipes bypass the registry's (0, 2) guard exactly like the reference test)
    proj = Recipe(base=RR, omega=0.0, omega_bulk_ho=0.0)
    for _ in range(10):
        f0 = near_eq(oracle, rng, 1.0, [0.02, 0.03, -0.01], 1e-2, q)
        once = apply(oracle, proj, f0, q)
        twice = apply(oracle, proj, once, q)
        assert near(twice, once, 1e-11)
        assert near(pi_neq(oracle, once, q), pi_neq(oracle, f0, q), 1e-10)
        assert near(moments(once, q), moments(f0, q), 1e-12)
    # RR ~ BGK near equilibrium at small velocity (test_collision.cpp:167-180)
    w = descriptor(q)[1]
    f = oracle.equilibrium(q, 2, 1.0, [1e-3, 5e-4, 0.0]) + rng.uniform(-1e-8, 1e-8, q)
    a = apply(oracle, Recipe(base=RR, omega=1.5), f, q)
    b = apply(oracle, Recipe(base=BGK, omega=1.5), f, q)
    # D3Q27 carries more non-hydrodynamic modes than the regularized basis, so
    # the filtered 1e-8 noise shows up relative to the 1/216 corner weights.
    assert np.all(np.abs(a - b) / (np.abs(b) + w) <= (1e-6 if q == 19 else 1e-5))


def test_smagorinsky_closed_form(oracle):  # test_collision.cpp:182-212
    # omega_eff is observable through BGK: f' = f - om_eff (f - feq)
    pi_xy = 3e-4
    f = oracle.equilibrium(19, 2, 1.0, [0, 0, 0]) + W19 * 4.5 * 2.0 * C19[:, 0] * C19[:, 1] * pi_xy
    om0, cs = 1.7, 0.16
    q_norm = math.sqrt(2.0 * (2.0 * pi_xy * pi_xy))
    tau0 = 1 / om0
    tau = 0.5 * (tau0 + math.sqrt(tau0 * tau0 + 2 * cs * cs * q_norm / (1.0 / 9.0)))
    out = apply(oracle, Recipe(base=BGK, omega=om0, has_les=True, smagorinsky_c=cs), f)
    m = moments(f)
    feq = oracle.equilibrium(19, 2, m[0], m[1:])
    om_eff = np.median((f - out)[f != feq] / (f - feq)[f != feq])
    assert near(om_eff, 1 / tau, 1e-10) and om_eff <= om0
    # laminar limit: C = 0 is plain BGK
    assert np.array_equal(apply(oracle, Recipe(base=BGK, omega=1.6, has_les=True, smagorinsky_c=0.0), f),
                          apply(oracle, Recipe(base=BGK, omega=1.6), f))


@pytest.mark.parametrize("q", [19, 27])
def test_conservation_random(oracle, q):  # test_collision.cpp:214-228
    rng = np.random.default_rng(31)
    for _ in range(25):
        f0 = rng.uniform(-0.02, 0.02, q)
        m0 = moments(f0, q)
        for r, tol in ((Recipe(base=BGK, omega=1.7), 1e-13),
                       (Recipe(base=TRT, omega=1.2), 1e-13),
                       (Recipe(base=RR, omega=1.9), 1e-12)):
            assert near(moments(apply(oracle, r, f0, q), q), m0, tol)


# --------------------------------------------------------------- boundaries
def test_bounce_back(oracle):  # test_boundaries.cpp:30-61
    rng = np.random.default_rng(41)
    f0 = rng.uniform(-0.05, 0.05, 19)
    f = apply(oracle, Recipe(kind=BB), f0)
    assert np.array_equal(f, f0[OPP19])
    assert np.array_equal(apply(oracle, Recipe(kind=BB), f), f0)
    assert np.array_equal(apply(oracle, Recipe(kind=MBB, wall_velocity=(0, 0, 0)), f0), f)
    assert np.array_equal(apply(oracle, Recipe(kind=NODYN), f0), f0)


def test_moving_bounce_back_ladd(oracle):  # test_boundaries.cpp:63-88
    rng = np.random.default_rng(47)
    uw = 0.1 / math.sqrt(3.0)
    f0 = rng.uniform(-0.05, 0.05, 19)
    f = apply(oracle, Recipe(kind=MBB, wall_velocity=(uw, 0, 0)), f0)
    assert near(f, f0[OPP19] + 2 * W19 * 3 * C19[:, 0] * uw, 1e-14)


def test_regularized_velocity_and_pressure(oracle):  # test_boundaries.cpp:90-129
    u_in = (0.02, 0.0, 0.0)
    fe = oracle.equilibrium(19, 2, 1.0, u_in)
    r = Recipe(base=BGK, omega=1.0, has_regularized=True, reg_axis=0, reg_orient=1, wall_velocity=u_in)
    assert near(apply(oracle, r, fe), fe, 1e-12)
    f = oracle.equilibrium(19, 2, 1.004, (0.03, 0, 0))
    out = apply(oracle, Recipe(base=BGK, omega=1.0, has_regularized=True, reg_orient=1,
                               wall_velocity=(0.03, 0, 0)), f)
    m = moments(out)
    assert near(m[0], 1.004, 1e-12) and near(m[1], 0.03, 1e-12)
    f = oracle.equilibrium(19, 2, 1.002, (0.015, 0, 0))
    out = apply(oracle, Recipe(base=BGK, omega=1.0, has_regularized=True, reg_is_pressure=True,
                               reg_orient=1, target_rho=1.002), f)
    m = moments(out)
    assert near(m[0], 1.002, 1e-12) and abs(m[1] - 0.015) < 5e-3 * (1 + 0.015)


# --------------------------------------------------------------- lattice level
def test_pulse_translation(oracle):  # test_reference_lattice.cpp:35-55
    n = 6
    for i in range(1, 19):
        f = np.zeros((19, n, n, n))
        f[i, 2, 2, 2] = 1.0
        r = Recipe(base=BGK, omega=0.0)  # omega = 0: pure streaming
        oracle.step(19, (n, n, n), (1, 1, 1), [r], np.zeros(n ** 3, np.int32), f.reshape(-1), 1)
        cx, cy, cz = C19[i]
        g = np.zeros_like(f)
        g[i, (2 + cz) % n, (2 + cy) % n, (2 + cx) % n] = 1.0
        assert np.array_equal(f, g)


def test_mass_conservation_periodic(oracle):  # test_reference_lattice.cpp:113-134
    case = Case(kind="tgv", L=12, Re=100.0, Ma=0.1, collision=BGK)
    dims, per, rec, slot = case.setup()
    f = oracle.initial_state(case, np.float64)
    m0 = f.sum()
    oracle.step(19, dims, per, rec, slot, f, 300)
    assert abs(f.sum() - m0) <= 1e-12 * max(1.0, abs(m0)) + 1e-12


def test_thread_count_bit_identity(oracle):  # test_accelerated.cpp:285-300
    case = Case(kind="cavity", L=16, Re=100.0, Ma=0.1, collision=TRT)
    a = oracle.run_case(case, np.float64, 30, nthreads=1)
    b = oracle.run_case(case, np.float64, 30, nthreads=5)
    assert np.array_equal(a, b)


# --------------------------------------------------------------- vs the reference
FAST_GOLDEN = [k for k, s in CASES.items() if s["steps"] * (s.get("L", 16) ** 3) <= 4e7]


@pytest.mark.parametrize("name", FAST_GOLDEN)
def test_oracle_matches_reference_golden(oracle, golden, name):
    """The oracle reproduces the committed hash of the reference's output bit for bit."""
    spec = CASES[name]
    case = make_case(spec)
    dt = np.float64 if spec["bits"] == 64 else np.float32
    out = oracle.run_case(case, dt, spec["steps"]).astype(np.float64)
    g = golden[name]
    assert np.array_equal(out[g["sample_index"]], np.asarray(g["sample"]))
    assert canonical_hash(out) == g["sha256"]


def test_case_tags_match_reference(reference):
    """The oracle's case generators assign the reference's chains cell by cell."""
    for case in (Case(kind="cavity", L=16),
                 Case(kind="porous", L=16, Ma=0.01, collision=TRT, plate_layers=6, upstream=4, downstream=4),
                 make_case(CASES["sphere48_trt_f64_c4"])):
        tags, models = reference.tags(case)
        _, _, rec, slot = case.setup()
        names = [r.chain_string() for r in rec]
        srt = sorted(set(names))
        assert models == srt
        mine = np.asarray([srt.index(n) for n in names])[slot]
        assert np.array_equal(tags, mine)


def test_kernels_bitwise_vs_reference(oracle, reference):
    """Every chain kind, both precisions: oracle == ChainRecipe<T>::apply bit for bit."""
    rng = np.random.default_rng(7)
    f = oracle.equilibrium(19, 2, 1.01, [0.03, -0.02, 0.04])[None, :] + rng.uniform(-2e-3, 2e-3, (64, 19))
    recipes = [
        Recipe(base=BGK, omega=1.7), Recipe(base=TRT, omega=1.3, lambda_=0.2),
        Recipe(base=RR, omega=1.9, omega_bulk_ho=1.1),
        Recipe(base=BGK, omega=1.6, has_les=True, smagorinsky_c=0.16),
        Recipe(base=TRT, omega=1.6, has_les=True, smagorinsky_c=0.12),
        Recipe(base=RR, omega=1.8, has_les=True, smagorinsky_c=0.1),
        Recipe(kind=BB), Recipe(kind=NODYN), Recipe(kind=MBB, wall_velocity=(0.05, -0.01, 0.02)),
        Recipe(base=TRT, omega=1.0, has_regularized=True, reg_axis=0, reg_orient=1, wall_velocity=(0.01, 0, 0)),
        Recipe(base=RR, omega=1.2, has_regularized=True, reg_axis=1, reg_orient=-1, wall_velocity=(0, 0.02, 0.01)),
        Recipe(base=BGK, omega=1.1, has_regularized=True, reg_is_pressure=True, reg_axis=2, reg_orient=1,
               target_rho=1.003),
        Recipe(base=TRT, omega=0.9, has_regularized=True, reg_is_pressure=True, reg_axis=0, reg_orient=-1,
               target_rho=0.998),
    ]
    for r in recipes:
        for bits, dt in ((64, np.float64), (32, np.float32)):
            mine = oracle.apply(19, r, f.astype(dt)).astype(np.float64)
            ref = reference.apply_chain(r.chain_string(), r.params(), bits, f.astype(dt).astype(np.float64))
            assert np.array_equal(mine, ref), (r.chain_string(), bits)


@pytest.mark.parametrize("name", ["tgv16_bgk_f64", "tgv12_bgk_f32", "cavity24_rr_f64",
                                  "plates16_trt_pres_f32", "tgv24_smag_trt_f32"])
def test_oracle_vs_reference_live(oracle, reference, name):
    spec = CASES[name]
    case = make_case(spec)
    dt = np.float64 if spec["bits"] == 64 else np.float32
    a = oracle.run_case(case, dt, spec["steps"]).astype(np.float64)
    b = reference.run_case(case, spec["bits"], spec["steps"], grid=(1, 1, 2), workers=2)
    assert np.array_equal(a, b)
