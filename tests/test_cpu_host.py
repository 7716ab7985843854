"""CPU-side checks of the product: the C-ABI library loads and exports every
symbol include/pardyn_c.h declares (no compute calls without a GPU), the
product-side workload generator reproduces the reference generators bit for
bit, host-side validation mirrors the reference's error behaviour, and the
batch partition is correct."""
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_symbols():
    with open(os.path.join(ROOT, "include", "pardyn_c.h")) as f:
        src = f.read()
    return sorted(set(re.findall(r"\b(pd_[a-z0-9_]+)\s*\(", src)))


def test_library_exports_every_header_symbol():
    from paper_1609_06779_b200 import _capi
    L = _capi.load()
    syms = header_symbols()
    assert len(syms) >= 15
    for s in syms:
        assert hasattr(L, s), s
    assert set(syms) == set(_capi.EXPORTS)
    assert L.pd_abi_version() == 1


def test_library_is_sm100a():
    """The in-tree .so carries sm_100a SASS (built by __graft_entry__.build)."""
    import subprocess
    from paper_1609_06779_b200 import _capi
    out = subprocess.run(["cuobjdump", "--list-elf", _capi.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_no_device_is_reported_not_hidden():
    """Without a GPU the product raises instead of falling back to a CPU path."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is visible")
    import paper_1609_06779_b200 as pd
    with pytest.raises(pd.CudaError):
        pd.Context(0)


def test_slot_messages_match_reference_strings():
    from paper_1609_06779_b200 import _capi as c
    assert c.slot_message(c.SLOT_DEGENERATE_ARTICULATION, 0, 7, 9) == \
        "degenerate articulation at joint 7: projected articulated inertia vanishes"
    assert c.slot_message(c.SLOT_OEE_SINGULAR_PIVOT, 1, 1, 3) == \
        "odd-even elimination: singular pivot block (round 1, block 1)"
    assert c.slot_message(c.SLOT_OEE_SINGULAR_FINAL, 3, 5, 8) == \
        "odd-even elimination: singular diagonal block after elimination (block 5)"
    assert c.slot_message(c.SLOT_BAD_MODEL, 0, 1, 3) == "spatial inertia: mass must be positive"
    assert c.slot_message(c.SLOT_BAD_SIZE, 0, 0, 4).startswith("forward dynamics: q, qdot and tau")
    assert c.slot_message(c.SLOT_JSI_NOT_SPD, 0, 0, 4).startswith("joint-space inertia is not positive definite")


def test_workload_generator_is_bit_exact(oracle):
    """pd_workload_* (product) == oracle == the pure-Python golden fixture."""
    import json
    from paper_1609_06779_b200 import workload as W
    cell = W.workload_seed(42, 32, 65536)
    assert cell == oracle.workload_seed(42, 32, 65536)
    assert np.array_equal(W.workload_chains(cell, 32, 64, g0=11), oracle.workload_chains(cell, 32, 64, g0=11))
    for a, b in zip(W.workload_inputs(cell, 32, 7, 2), oracle.workload_inputs(cell, 32, 7, 2)):
        assert np.array_equal(a, b)
    with open(os.path.join(ROOT, "tests", "golden", "workload.json")) as f:
        g = json.load(f)
    links = W.random_chain(3, 7)
    for i, rec in enumerate(g["random_chain_3_7"]):
        assert links[i, 0] == rec["mass"] and list(links[i, 13:19]) == rec["screw"]
        assert list(links[i, 28:31]) == rec["home_p"]


def test_batch_host_validation_without_gpu(oracle):
    """check_sizes runs on the host (forward_dynamics.cpp:19-31): invalid slots
    get the reference message, and a batch of only invalid slots never
    touches the device."""
    import paper_1609_06779_b200 as pd
    links, g = oracle.random_chain(3, 5)
    chain = pd.RobotChain.from_records(links, g)
    probs = [pd.FdProblem(chain, np.zeros(2), np.zeros(3), np.zeros(3)),
             pd.FdProblem(pd.RobotChain(), np.zeros(0), np.zeros(0), np.zeros(0))]
    res = pd.batch_forward_dynamics(probs, pd.FdAlgo.cfa)
    assert res[0].error == "forward dynamics: q, qdot and tau must each have one entry per joint (chain has 3)"
    assert res[1].error == "forward dynamics: chain has no links"
    with pytest.raises(pd.InvalidArgument):
        pd.forward_dynamics(chain, np.zeros(3), np.zeros(3), np.zeros(4), pd.FdAlgo.abia)
    with pytest.raises(pd.InvalidArgument):
        pd.forward_dynamics(chain, np.zeros(3), np.zeros(3), np.zeros(3), 7)


def test_linkspec_record_roundtrip(oracle):
    import paper_1609_06779_b200 as pd
    links, g = oracle.random_chain(4, 9)
    chain = pd.RobotChain.from_records(links, g)
    assert np.array_equal(chain.to_records(), links)


@pytest.mark.parametrize("total,world", [(10, 3), (65536, 8), (5, 8), (1, 1), (0, 2)])
def test_shard_bounds_partition(total, world):
    from paper_1609_06779_b200.sharding import shard_bounds
    covered = []
    for r in range(world):
        b, e = shard_bounds(total, world, r)
        assert 0 <= b <= e <= total
        covered.extend(range(b, e))
    assert covered == list(range(total))


def test_reference_arm_maps_only_the_oracle():
    """bench.py --impl reference runs the reference's CPU path (the oracle)
    and never maps the product library: its process loads oracle/build/
    liboracle.so and no libpardyn*.so."""
    import subprocess
    import sys
    code = (
        "import runpy, sys, json\n"
        "sys.argv = ['bench.py', '--impl', 'reference', '--workload', 'c1', '--steps', '1', '--warmup', '0']\n"
        "runpy.run_path('bench.py', run_name='__main__')\n"
        "libs = sorted({l.split()[-1] for l in open('/proc/self/maps') if l.rstrip().endswith('.so')})\n"
        "print('LIBS', json.dumps([x for x in libs if 'repo' in x or 'pardyn' in x or 'oracle' in x]))\n")
    r = subprocess.run([sys.executable, "-c", code], cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    line = [l for l in r.stdout.splitlines() if l.startswith("LIBS ")][-1]
    import json
    libs = json.loads(line[5:])
    assert any(x.endswith("oracle/build/liboracle.so") for x in libs), libs
    assert not any("libpardyn" in x for x in libs), libs
    out = json.loads([l for l in r.stdout.splitlines() if l.startswith("{")][-1])
    assert out["impl"] == "reference" and out["cpu_baseline"]["kind"] == "port"
