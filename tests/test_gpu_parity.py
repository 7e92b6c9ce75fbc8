"""GPU parity tests: the CUDA path (through the C-ABI) against the CPU oracle on the same
seeded inputs.  Tolerances (BASELINE.json north_star): max|a_gpu - a_ref| / max|a_ref|
<= 1e-5 for complex64, <= 1e-12 for complex128; integer / index work bit-exact."""
import hashlib
import json
import math
import os

import numpy as np
import pytest

from oracle import densitymatrix as dm
from oracle import einsum_net as tn
from oracle import lightcone as lc
from oracle import statevector as sv
from synth import circuits as C

pytestmark = pytest.mark.gpu

T = pytest.importorskip("paper_2104_10523_b200.tnqvm")
TOL = {T.C64: 1e-5, T.C128: 1e-12}
GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def relerr(a, b):
    a, b = np.asarray(a).reshape(-1), np.asarray(b).reshape(-1)
    return float(np.max(np.abs(a - b)) / np.max(np.abs(b)))


@pytest.fixture(scope="module")
def ctx():
    import torch
    assert torch.cuda.is_available()
    c = T.Context(0)
    yield c
    c.close()


@pytest.mark.parametrize("dtype", [T.C128, T.C64])
def test_ghz_qft_all_amplitudes(ctx, dtype):
    """Config 1: GHZ_8 then QFT, all 256 amplitudes vs the closed form and O1."""
    ops = C.ghz_qft(8)
    p = T.Plan(T.Circuit.from_oplist(ops), list(range(8)), 1 << 30, dtype=dtype, restarts=8)
    v = ctx.amplitudes(p, [-1] * 8)
    k = np.arange(256)
    closed = (1 + np.exp(-2j * np.pi * k / 256)) / math.sqrt(512)
    assert relerr(v, closed) <= TOL[dtype]
    assert relerr(v, sv.evolve(ops)) <= TOL[dtype]


@pytest.mark.parametrize("dtype", [T.C128, T.C64])
def test_bell_and_cat_state(ctx, dtype):
    p = T.Plan(T.Circuit.from_oplist(C.bell()), [], 1 << 20, dtype=dtype, restarts=2)
    assert abs(ctx.amplitude(p, [1, 1]) - 1 / math.sqrt(2)) < 10 * TOL[dtype]
    assert abs(ctx.amplitude(p, [0, 1])) < 10 * TOL[dtype]
    cat = T.Circuit.from_oplist(C.cat_state(60))
    p = T.Plan(cat, [2, 47], 1 << 20, dtype=dtype, restarts=4)
    for other, ref in ((0, [1, 0, 0, 0]), (1, [0, 0, 0, 1])):
        bits = [other] * 60
        bits[2] = bits[47] = -1
        v = ctx.amplitudes(p, bits)
        assert relerr(v, np.array(ref) / math.sqrt(2)) <= TOL[dtype]


@pytest.mark.parametrize("dtype", [T.C128, T.C64])
@pytest.mark.parametrize("seed", range(3))
def test_random_circuits_vs_statevector(ctx, dtype, seed):
    ops = C.random_circuit(10, 12, seed)
    psi = sv.evolve(ops)
    c = T.Circuit.from_oplist(ops)
    p = T.Plan(c, [], 1 << 30, dtype=dtype, restarts=8)
    rng = np.random.default_rng(seed)
    got, ref = [], []
    for _ in range(4):
        bits = rng.integers(0, 2, size=10)
        got.append(ctx.amplitude(p, bits))
        ref.append(psi[sv.index_of(bits)])
    assert relerr(got, ref) <= TOL[dtype]
    p = T.Plan(c, [0, 4, 9], 1 << 30, dtype=dtype, restarts=8)
    bits = list(rng.integers(0, 2, size=10))
    for q in (0, 4, 9):
        bits[q] = -1
    assert relerr(ctx.amplitudes(p, bits), sv.amplitudes(psi, bits)) <= TOL[dtype]
    # the whole state (norm = 1, brute force over 2^10)
    p = T.Plan(c, list(range(10)), 1 << 30, dtype=dtype, restarts=8)
    v = ctx.amplitudes(p, [-1] * 10)
    assert relerr(v, psi) <= TOL[dtype]
    assert abs(np.sum(np.abs(v) ** 2) - 1) < 100 * TOL[dtype]


@pytest.mark.parametrize("dtype", [T.C64, T.C128])
def test_sliced_grid_vs_statevector_and_slices(ctx, dtype):
    """4x5 grid RQC m=10 (n=20), budget forcing slicing: amplitudes vs O1, and the
    per-slice values vs O3 on identical slice ids (plan JSON wires read as data)."""
    ops = C.grid_rqc(4, 5, 10, seed=1)
    psi = sv.evolve(ops)
    c = T.Circuit.from_oplist(ops)
    es = 8 if dtype == T.C64 else 16
    p = T.Plan(c, [], es << 9, dtype=dtype, restarts=16)
    info = p.info()
    assert info["n_sliced"] >= 2 and info["log2_max_intermediate"] <= 9
    bits = C.random_bitstring(20, 1000)
    a = ctx.amplitude(p, bits)
    assert relerr([a], [psi[sv.index_of(bits)]]) <= TOL[dtype]
    ids = [0, 1, info["n_slices"] // 2, info["n_slices"] - 1]
    got = ctx.eval_slices(p, bits, ids)[:, 0]
    ref = tn.slice_values(tn.ket_network(ops, bits), p.sliced_wires(), ids, restarts=4)
    assert relerr(got, ref) <= TOL[dtype]
    # open qubits + slicing
    p = T.Plan(c, [0, 7, 13], es << 10, dtype=dtype, restarts=16)
    b2 = list(bits)
    for q in (0, 7, 13):
        b2[q] = -1
    assert relerr(ctx.amplitudes(p, b2), sv.amplitudes(psi, b2)) <= TOL[dtype]


def test_sycamore53_slice_subset_vs_einsum(ctx):
    """53-qubit Sycamore-layout RQC (m=8): identical slice ids on GPU and in O3."""
    ops = C.sycamore53(8, seed=0)
    c = T.Circuit.from_oplist(ops)
    p = T.Plan(c, [], 8 << 22, restarts=32, min_slices=16)
    info = p.info()
    bits = C.random_bitstring(53, 1001)
    ids = [3, info["n_slices"] - 2]
    got = ctx.eval_slices(p, bits, ids)[:, 0]
    ref = tn.slice_values(tn.ket_network(ops, bits), p.sliced_wires(), ids, restarts=4, cap_elems=2 ** 25)
    assert relerr(got, ref) <= 1e-5
    pc = T.Plan(c, [], 16 << 22, restarts=32, min_slices=16, dtype=T.C128)
    got = ctx.eval_slices(pc, bits, ids)[:, 0]
    ref = tn.slice_values(tn.ket_network(ops, bits), pc.sliced_wires(), ids, restarts=4, cap_elems=2 ** 25)
    assert relerr(got, ref) <= 1e-12


@pytest.mark.parametrize("dtype", [T.C64, T.C128])
def test_batched_units_bit_identical(ctx, monkeypatch, dtype):
    """a9 batching changes no arithmetic: the same amplitude from a replayed CUDA graph, a
    direct launch sequence, and inside amplitude_batch (other batch widths: 16 slices x 1,
    x 3 bitstrings per launch) is bit-identical; and equal to the group sums of the slices
    evaluated through eval_slices (another unit set) within rounding of the network scalar."""
    ops = C.sycamore53(8, seed=0)
    c = T.Circuit.from_oplist(ops)
    p = T.Plan(c, [], (8 if dtype == T.C64 else 16) << 22, restarts=32, min_slices=16, dtype=dtype)
    n = p.info()["n_slices"]
    assert n >= 16
    rows = [list(C.random_bitstring(53, 1002 + i)) for i in range(3)]
    vals = []
    for graph in ("0", "1"):
        monkeypatch.setenv("TNQVM_GRAPH", graph)
        vals.append(ctx.amplitude(p, rows[0]))
        vals.append(ctx.amplitude(p, rows[0]))  # second call replays the captured graph
    monkeypatch.setenv("TNQVM_GRAPH", "1")
    batch = ctx.amplitude_batch(p, rows)
    vals.append(batch[0])
    assert all(v == vals[0] for v in vals), vals
    assert batch[1] == ctx.amplitude(p, rows[1]) and batch[2] == ctx.amplitude(p, rows[2])
    per = ctx.eval_slices(p, rows[0], list(range(n)))[:, 0]
    assert relerr([vals[0]], [np.sum(per)]) <= (1e-6 if dtype == T.C64 else 1e-13)
    # the same slices in another order and batch composition: identical per-slice values
    ids = [n - 1, 3, 0, 7]
    per2 = ctx.eval_slices(p, rows[0], ids)[:, 0]
    assert np.array_equal(per2, per[ids])


@pytest.mark.parametrize("world", [2, 4, 8])
def test_emulated_ranks_group_slots(ctx, world):
    """a10 on one GPU: rank r of `world` (a context without a communicator) evaluates only
    the slice groups g = r mod world.  Each group slot taken from its owner equals the
    1-GPU slot bit for bit, so the NCCL allreduce of zero-padded slots (x + 0 = x) gives the
    1-GPU result exactly; the combined amplitudes match the oracle (O1, state vector)."""
    ops = C.grid_rqc(4, 5, 10, seed=2)
    psi = sv.evolve(ops)
    c = T.Circuit.from_oplist(ops)
    for dtype in (T.C64, T.C128):
        p = T.Plan(c, [0, 19], (8 if dtype == T.C64 else 16) << 12, restarts=8, min_slices=16, dtype=dtype)
        bits = list(C.random_bitstring(20, 1003))
        bits[0] = bits[19] = -1
        ref1 = ctx.amplitudes(p, bits)
        slots1 = ctx.group_slots()
        combined = np.zeros_like(slots1)
        for r in range(world):
            cr = T.Context(0, r, world)  # emulated rank: no nccl_id
            cr.amplitudes(p, bits)
            sr = cr.group_slots()
            for g in range(8):
                if g % world == r:
                    combined[g] = sr[g]
                else:
                    assert not np.any(sr[g])
            cr.close()
        assert np.array_equal(combined, slots1)
        # the host finalisation (group sum in order, network scalar) of the combined slots
        scalar = ref1[np.argmax(np.abs(ref1))] / slots1.sum(axis=0)[np.argmax(np.abs(ref1))]
        assert relerr(combined.sum(axis=0) * scalar, ref1) <= 1e-15
        assert relerr(ref1, sv.amplitudes(psi, bits)) <= TOL[dtype]


def test_stale_plan_on_device(ctx):
    """§8(b): using a plan after its circuit changed returns TNQVM_ESTATE."""
    c = T.Circuit.from_oplist(C.bell())
    p = T.Plan(c, [], 1 << 20, restarts=2)
    assert abs(ctx.amplitude(p, [1, 1]) - 1 / math.sqrt(2)) < 1e-6
    c.apply_gate(C.H, [1])
    with pytest.raises(T.TnqvmError) as e:
        ctx.amplitude(p, [1, 1])
    assert e.value.code == T.ESTATE


def test_graph_replay_new_values(ctx, monkeypatch):
    """A captured evaluation replayed for other bitstrings (new leaf values, new network
    scalar from the idle qubits' absorbed boundaries) matches the state vector."""
    ops = C.grid_rqc(3, 4, 8, seed=5)
    ops.nq = 14  # qubits 12, 13: only 1-qubit gates -> bitstring-dependent network scalar
    ops.gate(C.H, 12)
    ops.gate(C.rx(0.7), 13)
    psi = sv.evolve(ops)
    c = T.Circuit.from_oplist(ops)
    p = T.Plan(c, [], 8 << 8, restarts=8, min_slices=4)
    monkeypatch.setenv("TNQVM_GRAPH", "1")
    for seed in range(6):
        bits = C.random_bitstring(14, 300 + seed)
        a = ctx.amplitude(p, bits)
        assert ctx.stats()["graph"] == 1
        assert relerr([a], [psi[sv.index_of(bits)]]) <= 1e-5


@pytest.mark.parametrize("dtype", [T.C64, T.C128])
def test_amplitude_batch(ctx, dtype):
    """tnqvm_amplitude_batch (two alternating leaf/result regions, host build of bitstring i
    overlapping the device work of i - 1): every value equals the single-call amplitude bit
    for bit and the state vector within the dtype's tolerance; odd and even batch sizes,
    a batch of 1, an empty batch, a bitstring-dependent network scalar, a sliced plan."""
    ops = C.grid_rqc(3, 4, 8, seed=7)
    ops.nq = 14  # qubits 12, 13: only 1-qubit gates -> bitstring-dependent network scalar
    ops.gate(C.H, 12)
    ops.gate(C.rx(0.3), 13)
    psi = sv.evolve(ops)
    c = T.Circuit.from_oplist(ops)
    es = 8 if dtype == T.C64 else 16
    p = T.Plan(c, [], es << 8, dtype=dtype, restarts=8, min_slices=4)
    rows = [C.random_bitstring(14, 700 + i) for i in range(7)]
    for nb in (7, 4, 1):
        got = ctx.amplitude_batch(p, rows[:nb])
        one = np.array([ctx.amplitude(p, r) for r in rows[:nb]])
        assert np.array_equal(got, one)
        assert relerr(got, [psi[sv.index_of(r)] for r in rows[:nb]]) <= TOL[dtype]
    assert ctx.amplitude_batch(p, []).shape == (0,)
    with pytest.raises(T.TnqvmError):
        ctx.amplitude_batch(p, [rows[0], [2] * 14])


def _noisy(nrows, ncols, cycles, seed):
    return C.noisy_grid_circuit(nrows, ncols, cycles, seed)


def test_noisy_vs_density_matrix(ctx):
    """Doubled network with Kraus tensors vs dense rho (3x3 grid, m=4, c128)."""
    ops = _noisy(3, 3, 4, 2)
    rho = dm.evolve(ops)
    c = T.Circuit.from_oplist(ops)
    p = T.Plan(c, [], 1 << 30, dtype=T.C128, restarts=8)
    bits = [0, 1, 1, 0, 0, 1, 0, 1, 1]
    v = ctx.amplitude(p, bits)
    assert relerr([v], [dm.probability(rho, bits)]) <= 1e-12
    assert abs(v.imag) < 1e-14 and v.real >= 0
    p = T.Plan(c, [2, 5], 1 << 30, dtype=T.C128, restarts=8)
    b2 = list(bits)
    b2[2] = b2[5] = -1
    assert relerr(ctx.amplitudes(p, b2), dm.block(rho, b2)) <= 1e-12
    terms = [(1.0, [(0, "Z")]), (0.5, [(4, "X"), (5, "Y")]), (-1.0, [(8, "Z"), (7, "Z")])]
    tot, per = ctx.expectation(c, terms, per_term=True, dtype=T.C128, restarts=8)
    tot_ref, per_ref = dm.expectation(rho, terms)
    assert relerr(per, per_ref) <= 1e-12
    assert abs(tot - tot_ref) < 1e-12


def test_noisy_20q_vs_einsum_and_trace(ctx):
    """Config-5 shape at reduced depth: 4x5 noisy grid (m=4), <b|rho|b> vs O3 on its own
    doubled network; Tr rho = 1 with cancellation off."""
    ops = _noisy(4, 5, 4, 0)
    c = T.Circuit.from_oplist(ops)
    p = T.Plan(c, [], 16 << 20, dtype=T.C128, restarts=16)
    bits = C.random_bitstring(20, 1002)
    v = ctx.amplitude(p, bits)
    ref = tn.noisy_block(ops, bits, restarts=4)
    assert relerr([v], [ref]) <= 1e-12
    tot = ctx.expectation(c, [(1.0, [])], dtype=T.C128, cancel_conjugates=0, restarts=8)
    assert abs(tot - 1) < 1e-12
    z0 = ctx.expectation(c, [(1.0, [(0, "Z")])], dtype=T.C128, restarts=8)
    z0_full = ctx.expectation(c, [(1.0, [(0, "Z")])], dtype=T.C128, cancel_conjugates=0, restarts=8)
    assert abs(z0 - z0_full) < 1e-12


def _cube_edges():
    return sorted((a, b) for a in range(8) for b in range(a + 1, 8) if bin(a ^ b).count("1") == 1)


@pytest.mark.parametrize("dtype", [T.C128, T.C64])
def test_qaoa_expectations(ctx, dtype):
    """p=1 closed form on a triangle-free 3-regular graph; config 4 (40q, p=2) vs O4."""
    edges = _cube_edges()
    g, b = 0.37, 0.81
    ops = C.qaoa_circuit(8, edges, [g], [b])
    terms = C.maxcut_terms(edges)
    tot, per = ctx.expectation(T.Circuit.from_oplist(ops), terms, per_term=True, dtype=dtype, restarts=8)
    ref = math.sin(4 * b) * math.sin(2 * g) * math.cos(2 * g) ** 2
    assert relerr(per, np.full(len(terms), ref)) <= 10 * TOL[dtype]
    ops, terms = C.qaoa40(0)
    tot, per = ctx.expectation(T.Circuit.from_oplist(ops), terms, per_term=True, dtype=dtype, restarts=8)
    ref_tot, ref_per = lc.expectation(ops, terms)
    assert relerr(per, ref_per) <= TOL[dtype]
    assert abs(tot - ref_tot) <= TOL[dtype] * 60
    assert abs(tot.imag) < 1e-6


def test_pure_expectation_vs_statevector(ctx):
    ops = C.random_circuit(9, 10, 7)
    psi = sv.evolve(ops)
    c = T.Circuit.from_oplist(ops)
    terms = [(1.0, [(0, "Z"), (1, "Z")]), (0.3, [(2, "X")]), (0.7, [(3, "Y"), (8, "X")]), (2.0, [])]
    for cancel in (1, 0):
        tot, per = ctx.expectation(c, terms, per_term=True, dtype=T.C128, cancel_conjugates=cancel, restarts=8)
        tot_ref, per_ref = sv.expectation(psi, 9, terms)
        assert relerr(per, per_ref) <= 1e-12
        assert abs(tot - tot_ref) < 1e-12


# ---------------------------------------------------------------------------
# single kernels vs plain PyTorch references
# ---------------------------------------------------------------------------


@pytest.mark.parametrize("dtype", [T.C64, T.C128])
@pytest.mark.parametrize("rank,seed", [(1, 0), (5, 1), (12, 2), (17, 3), (22, 4)])
def test_permute_kernel(ctx, dtype, rank, seed):
    import torch
    rng = np.random.default_rng(seed)
    perm = rng.permutation(rank)
    td = torch.complex64 if dtype == T.C64 else torch.complex128
    x = torch.randn((2,) * rank, dtype=td, device="cuda")
    y = torch.empty_like(x)
    ctx.permute(dtype, x.data_ptr(), y.data_ptr(), rank, perm)
    ref = x.permute(*[int(p) for p in perm]).contiguous()
    assert torch.equal(y, ref)  # bit-exact: a permute moves bytes


@pytest.mark.parametrize("N,K,M", [(128, 2, 8), (1000, 16, 4), (4096, 16, 16), (70001, 64, 32), (33, 256, 64),
                                   (5000, 2, 256), (2 ** 20, 16, 8), (300, 2048, 128), (128, 4096, 64),
                                   (2048, 512, 512), (2 ** 18, 128, 128),
                                   # CTA-pair (cta_group::2) shapes: ragged last pair, half-tile W^T rows 16..128
                                   (1000, 256, 256), (4224, 128, 32), (700, 1024, 16), (2 ** 17, 32, 512)])
def test_gemm_tcgen05_3xtf32(ctx, N, K, M):
    """N2: tcgen05 3xTF32 complex64 GEMM vs a complex128 reference; accuracy within 4x
    of torch complex64 (allow_tf32=False) and <= 1e-6 relative for K <= 2^10
    (SURVEY §8(d))."""
    import torch
    torch.backends.cuda.matmul.allow_tf32 = False
    g = torch.Generator(device="cuda").manual_seed(N * 7 + K * 3 + M)
    X = torch.randn((N, K), dtype=torch.complex64, device="cuda", generator=g)
    Y = torch.randn((K, M), dtype=torch.complex64, device="cuda", generator=g)
    Cm = torch.full((N, M), float("nan"), dtype=torch.complex64, device="cuda")
    ctx.gemm(T.C64, 2, X.data_ptr(), Y.data_ptr(), Cm.data_ptr(), N, K, M)
    ref = X.to(torch.complex128) @ Y.to(torch.complex128)
    scale = ref.abs().max()
    err = float((Cm.to(torch.complex128) - ref).abs().max() / scale)
    err32 = float(((X @ Y).to(torch.complex128) - ref).abs().max() / scale)
    print(f"tc N={N} K={K} M={M} err={err:.3e} fp32_err={err32:.3e}")
    # SURVEY 8(d) N2 bar: <= 4x torch complex64 (allow_tf32=False) and <= 1e-6 for K <= 2^10
    assert err <= 4 * err32, (err, err32)
    if K <= 1024:
        assert err <= 1e-6, err


_GATHER_LAYOUTS = [
    # X bits fastest-first (the program's gather steps; 'n' row bits, 'k' contracted bits), M bits
    ("k0 n0 n1 n2 n3 n4 k1 n5 k2 n6 n7 n8 n9 k3 k4 n10 n11 n12 n13", 6),   # C2 op13-like: TMA box, TMEM-A
    ("k0 n0 n1 n2 n3 n4 n5 n6 k1 n7 k2 n8 n9 k3 k4 k5 k6 n10 n11", 7),      # op14-like: box, CTA pairs
    ("k0 k1 k2 n0 n1 n2 n3 n4 n5 n6 n7 n8 k3 k4 n9 k5 n10 n11 n12", 6),      # op9-like: box, 4-way banks
    ("k0 k1 k2 n0 n1 n2 n3 n4 k3 k4 n5 n6 n7 n8 k5 n9 n10 k6 n11 n12", 6),   # op15-like
    ("k0 n0 n7 n1 n8 n2 n9 n3 n10 n4 n11 n5 n12 n6 k1 k2 k3 k4", 5),         # > 5 runs: cp.async gather
    ("k0 n0 n1 k1 n2 n3 n4 k2 n5 n6 n7 n8 n9", 4),                           # K = 8: cp.async gather
    ("k0 n0 k1 n1 k2 n2 k3 n3 n4 k4 n5", 6),                                 # N = 64 rows: cp.async
    ("k0 n0 n1 n2 n3 n4 n5 n6 k1 k2 k3 n7 n8 n9 n10 n11 n12 n13", 1),        # narrow M
]


@pytest.mark.parametrize("order,nm", _GATHER_LAYOUTS)
def test_gemm_gather_layouts(ctx, order, nm):
    """N2 gather steps (X's fastest mode contracted, its other modes anywhere): the tcgen05
    kernel through the TMA-box producer (tile bits in <= 5 contiguous runs) or the cp.async
    fallback, against a complex128 reference on the same X; the N2 bar (4x / 1e-6)."""
    import torch
    torch.backends.cuda.matmul.allow_tf32 = False
    bits = order.split()
    nn = sum(b[0] == "n" for b in bits)
    nk = sum(b[0] == "k" for b in bits)
    N, K, M = 2 ** nn, 2 ** nk, 2 ** nm
    pos = {b: i for i, b in enumerate(bits)}
    sxn = [2 ** pos[f"n{i}"] for i in range(nn)]
    sxk = [2 ** pos[f"k{i}"] for i in range(nk)]
    g = torch.Generator(device="cuda").manual_seed(nn * 131 + nk * 7 + nm)
    Xf = torch.randn(N * K, dtype=torch.complex64, device="cuda", generator=g)
    Y = torch.randn((K, M), dtype=torch.complex64, device="cuda", generator=g)
    Cm = torch.full((N, M), float("nan"), dtype=torch.complex64, device="cuda")
    ctx.gemm_gather(T.C64, Xf.data_ptr(), Y.data_ptr(), Cm.data_ptr(), nn, nk, nm, sxn, sxk)
    slow = list(reversed(bits))
    perm = [slow.index(f"n{i}") for i in reversed(range(nn))] + [slow.index(f"k{i}") for i in reversed(range(nk))]
    Xm = Xf.view((2,) * (nn + nk)).permute(perm).reshape(N, K)
    ref = Xm.to(torch.complex128) @ Y.to(torch.complex128)
    scale = ref.abs().max()
    err = float((Cm.to(torch.complex128) - ref).abs().max() / scale)
    err32 = float(((Xm @ Y).to(torch.complex128) - ref).abs().max() / scale)
    assert err <= 4 * err32 and err <= 1e-6, (err, err32)


@pytest.mark.parametrize("N,K,M", [(64, 2, 4), (1000, 16, 8), (70001, 64, 32), (33, 256, 64), (300, 2048, 128),
                                   (4096, 512, 512), (16, 2 ** 16, 8),
                                   # 128-row tiles: 64 real columns, and the 32-column tile for M <= 16
                                   (2 ** 18, 64, 64), (2 ** 20, 16, 16), (2 ** 19, 64, 8), (300001, 16, 2)])
def test_gemm_dmma_c128(ctx, N, K, M):
    """N3: FP64 DMMA complex128 GEMM vs complex128 torch.matmul (<= 1e-13 relative)."""
    import torch
    g = torch.Generator(device="cuda").manual_seed(N + 3 * K + 7 * M)
    X = torch.randn((N, K), dtype=torch.complex128, device="cuda", generator=g)
    Y = torch.randn((K, M), dtype=torch.complex128, device="cuda", generator=g)
    Cm = torch.full((N, M), float("nan"), dtype=torch.complex128, device="cuda")
    ctx.gemm(T.C128, 2, X.data_ptr(), Y.data_ptr(), Cm.data_ptr(), N, K, M)
    ref = X @ Y
    err = float((Cm - ref).abs().max() / ref.abs().max())
    assert err <= 1e-13, err


@pytest.mark.parametrize("N,K,M", [(1, 1, 1), (1000, 4, 8), (4096, 16, 16), (70000, 64, 32), (33, 256, 64),
                                   (5000, 2, 256), (2 ** 20, 16, 4)])
@pytest.mark.parametrize("dtype", [T.C64, T.C128])
def test_gemm_simt_kernel(ctx, N, K, M, dtype):
    import torch
    td = torch.complex64 if dtype == T.C64 else torch.complex128
    g = torch.Generator(device="cuda").manual_seed(N + K + M)
    X = torch.randn((N, K), dtype=td, device="cuda", generator=g)
    Y = torch.randn((K, M), dtype=td, device="cuda", generator=g)
    Cm = torch.empty((N, M), dtype=td, device="cuda")
    ctx.gemm(dtype, 1, X.data_ptr(), Y.data_ptr(), Cm.data_ptr(), N, K, M)
    ref = (X.to(torch.complex128) @ Y.to(torch.complex128))
    err = (Cm.to(torch.complex128) - ref).abs().max() / ref.abs().max()
    assert float(err) <= (1e-5 if dtype == T.C64 else 1e-13)


@pytest.mark.parametrize("N,K,M", [(1, 2 ** 12, 1), (4, 2 ** 13, 2), (2, 2 ** 15, 8), (32, 2 ** 14, 8),
                                   (64, 2 ** 16, 64), (16, 2 ** 20, 4), (64, 2, 64), (8, 16, 32),
                                   (32, 2 ** 13, 4), (8, 2 ** 13, 4),  # K groups 2 and 8 (complex64)
                                   # complex64 lane kernel: 16 and 8 outputs per lane, 2 and 4 r-groups per warp
                                   (16, 2 ** 12, 16), (4, 2 ** 16, 16), (32, 2 ** 18, 8), (2, 2 ** 14, 16)])
@pytest.mark.parametrize("dtype", [T.C64, T.C128])
def test_gemm_splitk_strided(ctx, N, K, M, dtype):
    """Split-K (tiny / small outputs over long K; shared-memory tile gather, register
    blocks, fp64 partials) vs complex128 torch.matmul; the K < tile case included."""
    import torch
    td = torch.complex64 if dtype == T.C64 else torch.complex128
    g = torch.Generator(device="cuda").manual_seed(N + 5 * K + 11 * M)
    X = torch.randn((N, K), dtype=td, device="cuda", generator=g)
    Y = torch.randn((K, M), dtype=td, device="cuda", generator=g)
    Cm = torch.full((N, M), float("nan"), dtype=td, device="cuda")
    ctx.gemm(dtype, 3, X.data_ptr(), Y.data_ptr(), Cm.data_ptr(), N, K, M)
    ref = X.to(torch.complex128) @ Y.to(torch.complex128)
    err = float((Cm.to(torch.complex128) - ref).abs().max() / ref.abs().max())
    assert err <= (1e-5 if dtype == T.C64 else 1e-13), err


def _golden_c2():
    rows = []
    for line in open(os.path.join(GOLDEN, "c2_amplitudes.txt")):
        if line.startswith("#") or not line.strip():
            continue
        name, bits, re_, im_, _ = line.split()
        rows.append(([int(ch) for ch in bits], complex(float(re_), float(im_))))
    return rows


def test_c2_bench_config_full_size(ctx):
    """Config 2 at full size, in bench.py's configuration (Sycamore-53 m=10, circuit seed 0,
    16 GiB budget, 4096 restarts, planner seed 2, min_slices 8, B200 time-model objective): the WHOLE
    amplitude of the product path (all 8 slices batched, CUDA graph) vs O3's full
    contraction of its own network (tests/golden/c2_amplitudes.txt, written by
    tools/gen_goldens.py c2 from oracle/ only) for 2 bitstrings, <= 1e-5 relative
    (north_star complex64); and the product amplitude equal to the sum of its per-slice
    values (eval_slices: another batch composition)."""
    import bench  # the bench's own plan options (tests/test_host.py keeps them in sync with the goldens)
    ops = C.sycamore53(bench.CYCLES, bench.CIRCUIT_SEED)
    c = T.Circuit.from_oplist(ops)
    p = T.Plan(c, [], bench.BUDGET_BYTES, seed=bench.PLAN_SEED, restarts=bench.RESTARTS, dtype=T.C64,
               min_slices=bench.MIN_SLICES, cost_model=1)
    info = p.info()
    assert info["n_slices"] == 8
    for bits, ref in _golden_c2():
        amp = ctx.amplitude(p, bits)
        err = abs(amp - ref) / abs(ref)
        print(f"C2 whole amplitude rel err {err:.2e} (|a| 2^{math.log2(abs(ref)):.1f})")
        assert err <= 1e-5, (amp, ref)
        per = ctx.eval_slices(p, bits, list(range(info["n_slices"])))[:, 0]
        assert abs(amp - per.sum()) <= 1e-12 * np.abs(per).max()


def _golden_slices(name):
    d = json.load(open(os.path.join(GOLDEN, f"{name}_slices.json")))
    plan_cfg = json.load(open(os.path.join(GOLDEN, f"{name}_sliced_wires.json")))
    vals = np.array([[complex(re_, im_) for re_, im_ in v] for v in d["values"]])
    return plan_cfg, d, vals


def test_c3_slice_subset_vs_oracle(ctx):
    """Config-3 shape at full size (Sycamore-53 m=14, open qubits 0..5 -> 64-vectors)
    planned at a small budget (2^22 complex64 elements, 2^27 slices of ~2^32.5 MACs): two
    slices on the GPU vs O3 fixing the SAME wires of its own network (slice ids and wire
    names as data; tests/golden/c3_slices.json from tools/gen_goldens.py c3), the 64-vector
    <= 1e-5 relative (north_star complex64)."""
    cfg, d, ref = _golden_slices("c3")
    ops = C.sycamore53(cfg["cycles"], cfg["seed"])
    p = T.Plan(T.Circuit.from_oplist(ops), cfg["open"], cfg["budget"], restarts=cfg["restarts"],
               seed=cfg["plan_seed"], dtype=T.C64)
    assert hashlib.sha256(p.json().encode()).hexdigest() == d["plan_sha256"]  # the same plan (bit-exact)
    assert p.sliced_wires() == cfg["sliced"]
    bits = list(C.random_bitstring(53, 1004))
    for q in cfg["open"]:
        bits[q] = -1
    got = ctx.eval_slices(p, bits, d["slice_ids"])
    for i in range(len(d["slice_ids"])):
        assert relerr(got[i], ref[i]) <= 1e-5, i


def test_c5_noisy_m6_full_vs_oracle(ctx):
    """Config-5 shape (4x5 noisy grid, doubled network with depolarizing + amplitude-damping
    Kraus tensors, complex128) at m=6 in full: <b|rho|b> for 2 bitstrings and the 2x2 rho
    block of two open qubits vs O3 contracting its own doubled network (Eq.(3), P:L226-231,
    P:L252), <= 1e-12 relative (north_star complex128)."""
    ops = C.noisy_grid_circuit(4, 5, 6, 0)
    c = T.Circuit.from_oplist(ops)
    p = T.Plan(c, [], 16 << 24, dtype=T.C128, restarts=16)
    for seed in (1005, 1006):
        bits = C.random_bitstring(20, seed)
        v = ctx.amplitude(p, bits)
        ref = tn.noisy_block(ops, bits, restarts=4)
        assert relerr([v], [ref]) <= 1e-12
        assert v.real >= 0 and abs(v.imag) <= 1e-15
    p2 = T.Plan(c, [3, 11], 16 << 24, dtype=T.C128, restarts=16)
    bits = list(C.random_bitstring(20, 1007))
    bits[3] = bits[11] = -1
    assert relerr(ctx.amplitudes(p2, bits), tn.noisy_block(ops, bits, restarts=4)) <= 1e-12


def test_c5_noisy_m8_slices_vs_oracle(ctx):
    """Config 5 at its throughput depth (m=8) on two slices of a small-budget plan of the
    same doubled network (2^20 complex128 elements, 4096 slices): the GPU per-slice values
    vs O3 on the same slice ids (tests/golden/c5_slices.json), <= 1e-12 relative."""
    cfg, d, ref = _golden_slices("c5")
    ops = C.noisy_grid_circuit(cfg["rows"], cfg["cols"], cfg["cycles"], cfg["seed"])
    p = T.Plan(T.Circuit.from_oplist(ops), cfg["open"], cfg["budget"], restarts=cfg["restarts"],
               seed=cfg["plan_seed"], dtype=T.C128)
    assert hashlib.sha256(p.json().encode()).hexdigest() == d["plan_sha256"]
    bits = C.random_bitstring(20, 1005)
    got = ctx.eval_slices(p, bits, d["slice_ids"])[:, 0]
    assert relerr(got, ref[:, 0]) <= 1e-12
