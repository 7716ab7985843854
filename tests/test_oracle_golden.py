"""Pins the CPU oracle (oracle/) against the known answers the reference's own
tests define, stored as fixtures in tests/golden/ by
tests/golden/make_golden.py (pure Python, independent of the oracle)."""
import json
import os

import numpy as np
import pytest

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def load(name):
    with open(os.path.join(GOLDEN, name)) as f:
        return json.load(f)


def link(mass, com, inertia, screw=(0, 0, 1, 0, 0, 0), R=np.eye(3), p=(0, 0, 0)):
    return np.concatenate([[mass], com, np.asarray(inertia).ravel(), screw, np.asarray(R).ravel(), p])


def pendulum_chain(d):
    """oracles.hpp:299-309: joint about +z, gravity along -y."""
    links = np.array([link(d["mass"], [d["lc"], 0, 0], np.diag([0.11, 0.13, d["izz"]]))])
    return links, [0.0, -d["g"], 0.0]


def arm_chain(d):
    """oracles.hpp:327-347."""
    first = link(d["m1"], [d["lc1"], 0, 0], np.diag([0.05, 0.04, d["izz1"]]))
    second = link(d["m2"], [d["lc2"], 0, 0], np.diag([0.02, 0.03, d["izz2"]]), p=(-d["l1"], 0, 0))
    return np.array([first, second]), [0.0, -d["g"], 0.0]


@pytest.mark.parametrize("algo", ["jsiia", "abia", "cfa"])
def test_pendulum_forward_dynamics(oracle, algo):
    """test_fwddyn.cpp:105-122: every algorithm within 1e-8 * max(1, |qdd|)."""
    g = load("closed_form.json")
    links, grav = pendulum_chain(g["pendulum"])
    for s in g["pendulum_fd"]:
        got = oracle.forward_dynamics(algo, links, grav, [s["q"]], [s["qdot"]], [s["tau"]])[0]
        assert abs(got - s["qddot"]) < 1e-8 * max(1.0, abs(s["qddot"]))


def test_pendulum_inverse_dynamics(oracle):
    """test_invdyn.cpp:112-127."""
    g = load("closed_form.json")
    links, grav = pendulum_chain(g["pendulum"])
    for s in g["pendulum_id"]:
        got = oracle.inverse_dynamics(links, grav, [s["q"]], [s["qdot"]], [s["qddot"]])[0]
        assert abs(got - s["tau"]) < 1e-8 * max(1.0, abs(s["tau"]))


@pytest.mark.parametrize("algo", ["jsiia", "abia", "cfa"])
def test_arm_forward_dynamics(oracle, algo):
    """test_fwddyn.cpp:124-139: rel_gap <= 1e-8."""
    g = load("closed_form.json")
    links, grav = arm_chain(g["arm"])
    for s in g["arm_fd"]:
        got = oracle.forward_dynamics(algo, links, grav, s["q"], s["qdot"], s["tau"])
        want = np.array(s["qddot"])
        assert np.linalg.norm(got - want) / max(1.0, np.linalg.norm(want)) < 1e-8


def test_arm_inverse_dynamics(oracle):
    """test_invdyn.cpp:129-142."""
    g = load("closed_form.json")
    links, grav = arm_chain(g["arm"])
    for s in g["arm_id"]:
        got = oracle.inverse_dynamics(links, grav, s["q"], s["qdot"], s["qddot"])
        want = np.array(s["tau"])
        assert np.linalg.norm(got - want) / max(1.0, np.linalg.norm(want)) < 1e-8


def test_spec_kats(oracle):
    """SPEC.md examples: scan, bi-diagonal, OEE; test_oee.cpp:106-126 singular pivot."""
    k = load("spec_kat.json")
    out, rounds = oracle.scan_int64(k["scan_int"]["items"])
    assert list(out) == k["scan_int"]["expected"] and rounds == 2
    bd = k["bidiag_scalar"]
    x, _ = oracle.bidiag_solve(np.array(bd["coupling"]).reshape(-1, 1, 1), np.array(bd["rhs"]).reshape(-1, 1))
    assert np.allclose(x.ravel(), bd["expected"], rtol=0, atol=1e-15)
    oe = k["oee_2x1"]
    x, rounds = oracle.tridiag_solve(np.array(oe["diag"]).reshape(-1, 1, 1), np.array(oe["upper"]).reshape(-1, 1, 1),
                                     np.array(oe["rhs"]).reshape(-1, 1))
    assert np.allclose(x.ravel(), oe["expected"], atol=1e-15) and rounds == 1
    sg = k["oee_singular"]
    with pytest.raises(oracle.OracleError) as e:
        oracle.tridiag_solve(np.array(sg["diag"], float), np.array(sg["upper"], float), np.array(sg["rhs"], float))
    assert e.value.kind == "SingularBlockError"
    assert (e.value.round, e.value.index) == (sg["round"], sg["index"])
    assert "singular pivot" in str(e.value)


def test_rng_and_workload_seeds(oracle):
    """std::mt19937_64 check value; bench.cpp seeds and input streams."""
    w = load("workload.json")
    assert oracle.mt19937_64_nth(5489, 10000) == int(w["mt19937_64_seed5489_10000th"])
    assert oracle.mix(0) == int(w["mix_of_0"])
    assert oracle.workload_seed(42, 8, 1) == int(w["workload_seed_42_8_1"])
    assert oracle.workload_seed(42, 32, 65536) == int(w["workload_seed_42_32_65536"])
    cell = int(w["workload_seed_42_8_1"])
    for rep, key in ((0, "workload_inputs_c1_repeat0"), (5, "workload_inputs_c1_repeat5")):
        q, qd, dr = oracle.workload_inputs(cell, 8, 1, rep)
        gq, gqd, gdr = w[key][0]
        assert np.array_equal(q[0], gq) and np.array_equal(qd[0], gqd) and np.array_equal(dr[0], gdr)


@pytest.mark.parametrize("key,n,seed_key", [("random_chain_3_7", 3, None), ("random_chain_c1", 8, "chain_seed_g0")])
def test_random_chain_matches_golden(oracle, key, n, seed_key):
    """random_chain draw order (GCC right-to-left argument evaluation)."""
    w = load("workload.json")
    seed = 7 if seed_key is None else int(w[seed_key])
    links, grav = oracle.random_chain(n, seed)
    assert list(grav) == [0.0, 0.0, -9.81]
    for i, g in enumerate(w[key]):
        r = links[i]
        assert r[0] == g["mass"]
        assert list(r[1:4]) == g["com"]
        assert list(r[13:19]) == g["screw"]
        assert np.array_equal(r[19:28].reshape(3, 3), np.array(g["home_R"]))
        assert list(r[28:31]) == g["home_p"]
        I = r[4:13].reshape(3, 3)
        assert np.allclose(I, np.array(g["inertia"]), rtol=0, atol=1e-15)
        assert np.array_equal(I, I.T)
