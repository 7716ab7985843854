"""The pardyn drop-in C++ API (include/pardyn/pardyn.hpp, libpardyn.so over
the C-ABI): compiled and linked on CPU; run on the GPU as a C++ program that
reads like the reference's test_fwddyn.cpp (tests/cpp/test_dropin.cpp)."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "paper_1609_06779_b200", "lib")


def build(tmp_path, name="test_dropin"):
    exe = str(tmp_path / name)
    cmd = ["g++", "-O2", "-std=c++20", f"-I{ROOT}/include", os.path.join(ROOT, "tests", "cpp", name + ".cpp"),
           "-o", exe, f"-L{LIB}", "-lpardyn", "-lpardyn_b200", f"-Wl,-rpath,{LIB}"]
    subprocess.run(cmd, check=True, capture_output=True, text=True)
    return exe


def test_dropin_compiles_and_links(tmp_path):
    assert os.path.exists(os.path.join(LIB, "libpardyn.so"))
    build(tmp_path)
    build(tmp_path, "test_operators")


def test_reference_shaped_model_types_compile(tmp_path):
    """Caller code written against the reference's model types
    (model.hpp:17-30, spatial.hpp:15-150) compiles against the drop-in."""
    src = tmp_path / "caller.cpp"
    src.write_text(r"""
#include <pardyn/pardyn.hpp>
using namespace pardyn;
int main() {
  RobotChain chain;
  chain.gravity = Vec3(0.0, -9.81, 0.0);
  LinkSpec link;
  link.mass = 1.3;
  link.com = Vec3(0.45, 0.0, 0.0);
  link.inertia_rot = Mat3::Identity();
  link.joint_screw = Twist(Vec3::UnitZ(), Vec3::Zero());
  link.home_transform.rotation = Mat3::Identity();
  link.home_transform.translation = Vec3(0.1, 0.0, 0.0);
  chain.links.push_back(link);
  const SE3Transform t = screw_exp(link.joint_screw, 0.3) * link.home_transform;
  const AdjointMap ad = adjoint_of(t);
  const SpatialInertia J = spatial_inertia_from(link.mass, link.com, link.inertia_rot);
  const Wrench w = J.apply(ad.apply(Twist(Vec3::UnitX(), Vec3::Zero())));
  return (t.is_valid() && w.is_finite() && chain.size() == 1 && small_adjoint(Twist()).norm() == 0.0) ? 0 : 1;
}
""")
    exe = str(tmp_path / "caller")
    subprocess.run(["g++", "-O2", "-std=c++20", f"-I{ROOT}/include", str(src), "-o", exe, f"-L{LIB}", "-lpardyn",
                    "-lpardyn_b200", f"-Wl,-rpath,{LIB}"], check=True, capture_output=True, text=True)
    assert subprocess.run([exe]).returncode == 0  # host-side value algebra only: no device needed


def test_dropin_without_gpu_fails_loudly(tmp_path):
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is visible")
    r = subprocess.run([build(tmp_path)], capture_output=True, text=True)
    assert r.returncode != 0 and "cannot open CUDA device" in r.stderr


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["test_dropin", "test_operators"])
def test_dropin_cpp_suite_on_gpu(tmp_path, name):
    r = subprocess.run([build(tmp_path, name)], capture_output=True, text=True, timeout=600)
    print(r.stdout[-3000:])
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]
    assert "0 failure(s)" in r.stdout


def test_model_files_and_bench_csv_on_host(tmp_path, oracle):
    """validate_chain / load_chain / save_chain and the benchmark CSV of the
    drop-in (host-only code: runs without a GPU); the saved file follows the
    reference's JSON layout and holds the generator's exact values."""
    import json

    import numpy as np
    exe = str(tmp_path / "test_model_io")
    subprocess.run(["g++", "-O2", "-std=c++20", f"-I{ROOT}/include", os.path.join(ROOT, "tests", "cpp", "test_model_io.cpp"),
                    "-o", exe, f"-L{LIB}", "-lpardyn", "-lpardyn_b200", f"-Wl,-rpath,{LIB}"], check=True,
                   capture_output=True, text=True)
    r = subprocess.run([exe, str(tmp_path)], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0 and "0 failure(s)" in r.stdout, r.stdout + r.stderr
    doc = json.load(open(tmp_path / "m7.json"))
    assert list(doc) == ["n", "gravity", "links"] and doc["n"] == 7
    assert list(doc["links"][0]) == ["mass", "com", "inertia_rot", "joint_screw", "home_transform"]
    links, g = oracle.random_chain(7, 1234)
    for i, l in enumerate(doc["links"]):
        rec = np.concatenate([[l["mass"]], l["com"], l["inertia_rot"], l["joint_screw"],
                              l["home_transform"]["rotation"], l["home_transform"]["translation"]])
        assert np.array_equal(rec, links[i])


def test_python_model_files(tmp_path, oracle):
    import paper_1609_06779_b200 as pd
    links, g = oracle.random_chain(5, 99)
    chain = pd.RobotChain.from_records(links, g)
    pd.save_chain(chain, str(tmp_path / "c.json"))
    back = pd.load_chain(str(tmp_path / "c.json"))
    assert (back.to_records() == chain.to_records()).all() and (back.gravity == chain.gravity).all()
    bad = pd.RobotChain.from_records(links, g)
    bad.links[3].mass = -1.0
    with pytest.raises(pd.ModelError, match="^link 3: mass must be positive$"):
        pd.validate_chain(bad)
    (tmp_path / "b.json").write_text('{"n": 2, "gravity": [0, 0, -9.81], "links": []}')
    with pytest.raises(pd.ModelError, match=r"field 'n' \(= 2\) does not match the length of 'links' \(= 0\)"):
        pd.load_chain(str(tmp_path / "b.json"))


@pytest.mark.gpu
def test_bench_cli_on_gpu(tmp_path):
    """pardyn_bench (the reference's CLI flags and CSV) timing the GPU path."""
    out = tmp_path / "r.csv"
    exe = os.path.join(LIB, "pardyn_bench")
    r = subprocess.run([exe, "--mode", "link", "--algos", "jsiia,abia,cfa,invdyn", "--links", "8,40", "--repeats", "5",
                        "--out", str(out)], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr
    r2 = subprocess.run([exe, "--mode=group", "--algos=abia,cfa", "--links=16", "--groups=1,300", "--repeats=3",
                         f"--out={tmp_path / 'g.csv'}"], capture_output=True, text=True, timeout=600)
    assert r2.returncode == 0, r2.stdout + r2.stderr
    lines = out.read_text().splitlines()
    assert lines[0] == "algo,n_links,n_groups,repeats,worker_count,mean_us,stddev_us" and len(lines) == 9
    assert len((tmp_path / "g.csv").read_text().splitlines()) == 5
