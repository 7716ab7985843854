"""Generates tests/golden/*.json — known-answer vectors for this path.

The reference ships no data files and cannot be compiled here
(Eigen3 absent), so these fixtures are built from the reference's OWN
known-answer definitions, restated independently of the C++ oracle:

  * closed-form pendulum and planar 2-link arm (tests/support/oracles.hpp:293-382)
    on the exact TestRng streams the reference tests use
    (test_fwddyn.cpp:105-139, test_invdyn.cpp:112-142);
  * the SPEC.md known-answer examples (scan, bi-diagonal, OEE);
  * std::mt19937_64's standard check value (10000th draw of seed 5489);
  * the bench workload seeds and inputs (bench.cpp:42-70,350-383) and
    random_chain (model.cpp:26-56,157-185, GCC argument order), in pure Python.

Run: python tests/golden/make_golden.py   (rewrites the JSON files)
"""
import json
import math
import os

HERE = os.path.dirname(os.path.abspath(__file__))
M64 = (1 << 64) - 1


class MT19937_64:
    """std::mt19937_64 (pure Python)."""

    def __init__(self, seed):
        self.mt = [0] * 312
        self.mt[0] = seed & M64
        for i in range(1, 312):
            self.mt[i] = (6364136223846793005 * (self.mt[i - 1] ^ (self.mt[i - 1] >> 62)) + i) & M64
        self.i = 312

    def __call__(self):
        if self.i >= 312:
            for k in range(312):
                x = (self.mt[k] & 0xFFFFFFFF80000000) | (self.mt[(k + 1) % 312] & 0x7FFFFFFF)
                xa = x >> 1
                if x & 1:
                    xa ^= 0xB5026F5AA96619E9
                self.mt[k] = self.mt[(k + 156) % 312] ^ xa
            self.i = 0
        y = self.mt[self.i]
        self.i += 1
        y ^= (y >> 29) & 0x5555555555555555
        y ^= (y << 17) & 0x71D67FFFEDA60000
        y ^= (y << 37) & 0xFFF7EEE000000000
        y ^= y >> 43
        return y & M64


class TestRng:
    """oracles.hpp:39-62 / model.cpp Rng: top 53 bits to [0,1)."""

    def __init__(self, seed):
        self.e = MT19937_64(seed)

    def uniform(self, lo=0.0, hi=1.0):
        u = (self.e() >> 11) * 2.0 ** -53
        return lo + (hi - lo) * u

    def vector(self, n, lo=-1.0, hi=1.0):
        return [self.uniform(lo, hi) for _ in range(n)]


def mix(x):  # bench.cpp:42-47
    x = (x + 0x9E3779B97F4A7C15) & M64
    x = ((x ^ (x >> 30)) * 0xBF58476D1CE4E5B9) & M64
    x = ((x ^ (x >> 27)) * 0x94D049BB133111EB) & M64
    return x ^ (x >> 31)


def workload_seed(seed, n_links, n_groups):  # bench.cpp:350-355
    h = mix(seed)
    h = mix(h ^ n_links)
    return mix(h ^ ((n_groups << 20) & M64))


def workload_inputs(cell, n, groups, repeat):  # bench.cpp:368-383
    e = MT19937_64(mix(cell ^ ((0x5EED + repeat * 0x9E3779B97F4A7C15) & M64)))

    def sym():
        return 2.0 * ((e() >> 11) * 2.0 ** -53) - 1.0

    out = []
    for _ in range(groups):
        out.append(([sym() for _ in range(n)], [sym() for _ in range(n)], [sym() for _ in range(n)]))
    return out


def rotation(rng):  # model.cpp:40-52 + Eigen toRotationMatrix
    u1 = rng.uniform()
    a2 = rng.uniform(0.0, 2.0 * math.pi)
    a3 = rng.uniform(0.0, 2.0 * math.pi)
    s1, s2 = math.sqrt(1.0 - u1), math.sqrt(u1)
    w, x, y, z = s2 * math.cos(a3), s1 * math.sin(a2), s1 * math.cos(a2), s2 * math.sin(a3)
    tx, ty, tz = 2 * x, 2 * y, 2 * z
    twx, twy, twz = tx * w, ty * w, tz * w
    txx, txy, txz = tx * x, ty * x, tz * x
    tyy, tyz, tzz = ty * y, tz * y, tz * z
    return [[1 - (tyy + tzz), txy - twz, txz + twy], [txy + twz, 1 - (txx + tzz), tyz - twx],
            [txz - twy, tyz + twx, 1 - (txx + tyy)]]


def unit_vector(rng):  # model.cpp:32-37
    z = rng.uniform(-1.0, 1.0)
    phi = rng.uniform(0.0, 2.0 * math.pi)
    r = math.sqrt(max(0.0, 1.0 - z * z))
    return [r * math.cos(phi), r * math.sin(phi), z]


def random_chain_masses_screws(n, seed):
    """The parts of random_chain (model.cpp:157-185) that do not depend on
    Eigen's matrix-product summation order: masses, coms, screws, home
    rotations and translations (the inertia is summed by Eigen and only
    checked to tolerance)."""
    rng = TestRng(seed)
    links = []
    for _ in range(n):
        mass = rng.uniform(0.1, 10.0)
        cz, cy, cx = rng.uniform(-0.3, 0.3), rng.uniform(-0.3, 0.3), rng.uniform(-0.3, 0.3)
        axes = rotation(rng)
        mz, my, mx = rng.uniform(0.1, 1.0), rng.uniform(0.1, 1.0), rng.uniform(0.1, 1.0)
        d = [mx, my, mz]
        inertia = [[sum(axes[r][k] * d[k] * axes[c][k] for k in range(3)) for c in range(3)] for r in range(3)]
        screw = unit_vector(rng) + [0.0, 0.0, 0.0]
        R = rotation(rng)
        direction = unit_vector(rng)
        mag = rng.uniform(0.1, 1.0)
        links.append(dict(mass=mass, com=[cx, cy, cz], inertia=inertia, screw=screw, home_R=R,
                          home_p=[mag * v for v in direction]))
    return links


# ------------------------------------------------------------- closed forms
PEND = dict(mass=1.3, lc=0.45, izz=0.07, g=9.81)
ARM = dict(m1=1.8, m2=0.9, l1=0.6, lc1=0.35, lc2=0.25, izz1=0.06, izz2=0.025, g=9.81)


def pend_accel(q, tau):
    p = PEND
    return (tau - p["mass"] * p["g"] * p["lc"] * math.cos(q)) / (p["izz"] + p["mass"] * p["lc"] ** 2)


def pend_torque(q, qdd):
    p = PEND
    return (p["izz"] + p["mass"] * p["lc"] ** 2) * qdd + p["mass"] * p["g"] * p["lc"] * math.cos(q)


def arm_mass(q):
    a = ARM
    c2 = math.cos(q[1])
    m00 = a["izz1"] + a["izz2"] + a["m1"] * a["lc1"] ** 2 + a["m2"] * (
        a["l1"] ** 2 + a["lc2"] ** 2 + 2 * a["l1"] * a["lc2"] * c2)
    m01 = a["izz2"] + a["m2"] * (a["lc2"] ** 2 + a["l1"] * a["lc2"] * c2)
    m11 = a["izz2"] + a["m2"] * a["lc2"] ** 2
    return [[m00, m01], [m01, m11]]


def arm_bias(q, qd):
    a = ARM
    s2, c1, c12 = math.sin(q[1]), math.cos(q[0]), math.cos(q[0] + q[1])
    b0 = (-a["m2"] * a["l1"] * a["lc2"] * s2 * (2 * qd[0] * qd[1] + qd[1] ** 2)
          + (a["m1"] * a["lc1"] + a["m2"] * a["l1"]) * a["g"] * c1 + a["m2"] * a["lc2"] * a["g"] * c12)
    b1 = a["m2"] * a["l1"] * a["lc2"] * s2 * qd[0] ** 2 + a["m2"] * a["lc2"] * a["g"] * c12
    return [b0, b1]


def arm_accel(q, qd, tau):
    M = arm_mass(q)
    b = arm_bias(q, qd)
    r = [tau[0] - b[0], tau[1] - b[1]]
    det = M[0][0] * M[1][1] - M[0][1] * M[1][0]
    return [(M[1][1] * r[0] - M[0][1] * r[1]) / det, (-M[1][0] * r[0] + M[0][0] * r[1]) / det]


def arm_torque(q, qd, qdd):
    M = arm_mass(q)
    b = arm_bias(q, qd)
    return [M[0][0] * qdd[0] + M[0][1] * qdd[1] + b[0], M[1][0] * qdd[0] + M[1][1] * qdd[1] + b[1]]


def main():
    # pendulum FD: test_fwddyn.cpp:105-122 (TestRng(111), 50 trials, q, qdot, tau)
    rng = TestRng(111)
    pend_fd = []
    for _ in range(50):
        q, qd, tau = rng.uniform(-6, 6), rng.uniform(-4, 4), rng.uniform(-8, 8)
        pend_fd.append(dict(q=q, qdot=qd, tau=tau, qddot=pend_accel(q, tau)))
    # pendulum ID: test_invdyn.cpp:112-127 (TestRng(5150), 100 trials)
    rng = TestRng(5150)
    pend_id = []
    for _ in range(100):
        q, qd, qdd = rng.uniform(-6, 6), rng.uniform(-4, 4), rng.uniform(-10, 10)
        pend_id.append(dict(q=q, qdot=qd, qddot=qdd, tau=pend_torque(q, qdd)))
    # arm FD: test_fwddyn.cpp:124-139 (TestRng(222))
    rng = TestRng(222)
    arm_fd = []
    for _ in range(50):
        q, qd, tau = rng.vector(2, -6, 6), rng.vector(2, -4, 4), rng.vector(2, -8, 8)
        arm_fd.append(dict(q=q, qdot=qd, tau=tau, qddot=arm_accel(q, qd, tau)))
    # arm ID: test_invdyn.cpp:129-142 (TestRng(6006))
    rng = TestRng(6006)
    arm_id = []
    for _ in range(100):
        q, qd, qdd = rng.vector(2, -6, 6), rng.vector(2, -4, 4), rng.vector(2, -10, 10)
        arm_id.append(dict(q=q, qdot=qd, qddot=qdd, tau=arm_torque(q, qd, qdd)))
    with open(os.path.join(HERE, "closed_form.json"), "w") as f:
        json.dump(dict(source="tests/support/oracles.hpp:293-382; test_fwddyn.cpp:105-139; test_invdyn.cpp:112-142",
                       pendulum=PEND, arm=ARM, pendulum_fd=pend_fd, pendulum_id=pend_id, arm_fd=arm_fd,
                       arm_id=arm_id), f, indent=1)

    cell = workload_seed(42, 8, 1)
    wl = dict(
        source="bench.cpp:42-70,350-383; model.cpp:26-56,157-185",
        mt19937_64_seed5489_10000th=str(MT19937_64(5489).__class__ and _nth(5489, 10000)),
        mix_of_0=str(mix(0)),
        workload_seed_42_8_1=str(cell),
        workload_seed_42_32_65536=str(workload_seed(42, 32, 65536)),
        workload_inputs_c1_repeat0=workload_inputs(cell, 8, 1, 0),
        workload_inputs_c1_repeat5=workload_inputs(cell, 8, 1, 5),
        chain_seed_g0=str(mix(cell ^ (0xC0FFEE + 0))),
        random_chain_3_7=random_chain_masses_screws(3, 7),
        random_chain_c1=random_chain_masses_screws(8, mix(cell ^ (0xC0FFEE + 0))),
    )
    with open(os.path.join(HERE, "workload.json"), "w") as f:
        json.dump(wl, f, indent=1)

    spec = dict(
        source="SPEC.md scanblk / oee examples",
        scan_int=dict(items=[1, 2, 3, 4], expected=[1, 3, 6, 10]),
        bidiag_scalar=dict(coupling=[2.0, 2.0], rhs=[1.0, 0.0, 0.0], expected=[1.0, 2.0, 4.0]),
        oee_2x1=dict(diag=[2.0, 2.0], upper=[1.0], rhs=[3.0, 3.0], expected=[1.0, 1.0]),
        oee_singular=dict(n=3, B=2, diag=[[[1, 0], [0, 1]], [[0, 0], [0, 0]], [[1, 0], [0, 1]]],
                          upper=[[[0.1, 0], [0, 0.1]], [[0.1, 0], [0, 0.1]]], rhs=[[1, 1], [1, 1], [1, 1]],
                          round=1, index=1, source="test_oee.cpp:106-126"),
    )
    with open(os.path.join(HERE, "spec_kat.json"), "w") as f:
        json.dump(spec, f, indent=1)


def _nth(seed, n):
    e = MT19937_64(seed)
    v = 0
    for _ in range(n):
        v = e()
    return v


if __name__ == "__main__":
    main()
