"""GPU parity of the SURVEY §8(f) NEXT rows built on the same executor, against the oracle:
NEXT-2 expectation by wave-function slicing (Table 1) vs O1 / O7, and
NEXT-3 direct unbiased bit-string sampling (Table 1) vs O6 on the same uniforms."""
import math

import numpy as np
import pytest

from oracle import densitymatrix as dm
from oracle import sampling as smp
from oracle import statevector as sv
from synth import circuits as C

pytestmark = pytest.mark.gpu

T = pytest.importorskip("paper_2104_10523_b200.tnqvm")
TOL = {T.C64: 1e-5, T.C128: 1e-12}


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


TERMS10 = [(1.0, [(0, "Z"), (1, "Z")]), (0.5, [(2, "X"), (3, "Y")]), (-0.7, [(3, "Z"), (9, "Z")]),
           (0.25, [(4, "Y"), (8, "Z"), (6, "X")]), (2.0, [])]


@pytest.mark.parametrize("dtype", [T.C128, T.C64])
@pytest.mark.parametrize("rank_max", [4, 6, 10])
def test_wfslice_expectation_vs_statevector(ctx, dtype, rank_max):
    """NEXT-2: per-term <P_j> by wave-function slicing (2^(10 - rank_max) projected slices,
    internal slicing of each partial state vector at a small budget) vs the full state vector
    (O1) and the oracle's own slicing (O7)."""
    ops = C.random_circuit(10, 12, 4)
    psi = sv.evolve(ops)
    c = T.Circuit.from_oplist(ops)
    es = 8 if dtype == T.C64 else 16
    tot, per = ctx.expectation_wfslice(c, TERMS10, rank_max, es << max(8, rank_max), per_term=True, dtype=dtype,
                                       restarts=8)
    tot_ref, per_ref = sv.expectation(psi, 10, TERMS10)
    assert relerr(per, per_ref) <= TOL[dtype]
    assert abs(tot - tot_ref) <= 10 * TOL[dtype]
    _, per7 = smp.wf_slice_expectation(psi, 10, TERMS10, list(range(10)))
    assert relerr(per, per7) <= TOL[dtype]


def test_wfslice_qaoa_closed_form_and_errors(ctx):
    """QAOA p=1 on the cube graph: <Z_u Z_v> = sin4b sin2g cos^2 2g for every edge, with 4 of 8
    qubits projected; X / Y support larger than rank_max is EINVAL."""
    edges = sorted((a, b) for a in range(8) for b in range(a + 1, 8) if bin(a ^ b).count("1") == 1)
    g, b = 0.37, 0.81
    c = T.Circuit.from_oplist(C.qaoa_circuit(8, edges, [g], [b]))
    _, per = ctx.expectation_wfslice(c, C.maxcut_terms(edges), 4, 16 << 20, per_term=True, dtype=T.C128, restarts=4)
    ref = math.sin(4 * b) * math.sin(2 * g) * math.cos(2 * g) ** 2
    assert np.max(np.abs(per - ref)) <= 1e-12
    with pytest.raises(T.TnqvmError) as e:
        ctx.expectation_wfslice(c, [(1.0, [(0, "X"), (1, "X"), (2, "Y")])], 2, 16 << 20)
    assert e.value.code == T.EINVAL


def test_wfslice_emulated_ranks_partition(ctx):
    """Projected-bitstring groups split over emulated ranks: the per-rank partial values add
    up to the 1-rank value (each group is evaluated by exactly one rank)."""
    ops = C.random_circuit(9, 10, 6)
    c = T.Circuit.from_oplist(ops)
    terms = [(1.0, [(0, "Z"), (5, "Z")]), (0.5, [(1, "X")])]
    _, ref = ctx.expectation_wfslice(c, terms, 4, 16 << 10, per_term=True, dtype=T.C128, restarts=4)
    acc = np.zeros(2, dtype=complex)
    for r in range(4):
        cr = T.Context(0, r, 4)
        _, pr = cr.expectation_wfslice(c, terms, 4, 16 << 10, per_term=True, dtype=T.C128, restarts=4)
        acc += pr
        cr.close()
    assert relerr(acc, ref) <= 1e-13


def _safe_uniforms(probs, n, seed):
    cum = np.cumsum(probs)
    rng = np.random.default_rng(seed)
    return [u for u in rng.random(4 * n) if np.min(np.abs(cum - u)) > 1e-7][:n]


@pytest.mark.parametrize("block", [1, 2, 3])
def test_sampling_vs_oracle(ctx, block):
    """NEXT-3: 40 shots of a 9-qubit random circuit (complex128) from the same uniforms as
    the oracle's sequential sampler (O6, exact marginals of |psi|^2): identical bitstrings,
    and the returned probabilities equal |psi_b|^2."""
    ops = C.random_circuit(9, 10, 9)
    probs = smp.probabilities(sv.evolve(ops))
    us = _safe_uniforms(probs, 40, block)
    bits, p = ctx.sample(T.Circuit.from_oplist(ops), us, block=block, dtype=T.C128, restarts=4)
    ref = smp.sample(probs, 9, us, block)
    assert np.array_equal(bits, ref)
    assert relerr(p, [probs[sv.index_of(r)] for r in ref]) <= 1e-12


def test_sampling_noisy_and_ghz(ctx):
    """Noisy circuit (doubled network with Kraus tensors): samples from diag(rho) (O2 + O6);
    GHZ_12 gives only 0^12 / 1^12, split at u = 1/2."""
    ops = C.noisy_grid_circuit(3, 3, 3, 1)
    probs = np.real(np.diag(dm.as_matrix(dm.evolve(ops))))
    us = _safe_uniforms(probs, 24, 3)
    bits, _ = ctx.sample(T.Circuit.from_oplist(ops), us, block=2, dtype=T.C128, restarts=4)
    assert np.array_equal(bits, smp.sample(probs, 9, us, 2))
    g = T.Circuit.from_oplist(C.ghz(12))
    bits, p = ctx.sample(g, [0.1, 0.49, 0.51, 0.9], block=4, dtype=T.C64, restarts=4)
    assert [list(r) for r in bits] == [[0] * 12] * 2 + [[1] * 12] * 2
    assert np.max(np.abs(p - 0.5)) <= 1e-6


def test_plan_autotune_picks_a_measured_plan(ctx):
    """NEXT-1 plan selection by measured cost (tnqvm_plan_autotune): the returned plan is the
    plan of the seed with the smallest measured time (byte-identical plan JSON), and its
    amplitudes equal those of another seed's plan (a different contraction order) and the
    state vector's (O1) on a 20-qubit circuit."""
    ops = C.grid_rqc(4, 5, 8, 3)
    circ = T.Circuit.from_oplist(ops)
    rows = [list(C.random_bitstring(20, 70 + i)) for i in range(3)]
    seeds = [0, 1, 2]
    plan, ms = ctx.autotune_plan(circ, 1 << 24, seeds, rows, reps=2, restarts=16, dtype=T.C128, min_slices=4)
    assert len(ms) == 3 and all(m > 0 for m in ms)
    win = seeds[int(np.argmin(ms))]
    ref_plan = T.Plan(circ, [], 1 << 24, seed=win, restarts=16, dtype=T.C128, min_slices=4)
    assert plan.json() == ref_plan.json()
    other = T.Plan(circ, [], 1 << 24, seed=seeds[(seeds.index(win) + 1) % 3], restarts=16, dtype=T.C128, min_slices=4)
    a = ctx.amplitude_batch(plan, rows)
    b = ctx.amplitude_batch(other, rows)
    psi = sv.evolve(ops)
    ref = [sv.amplitude(psi, r) for r in rows]
    assert relerr(a, ref) <= 1e-12 and relerr(b, ref) <= 1e-12
