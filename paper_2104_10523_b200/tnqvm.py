"""Thin ctypes binding of libtnqvm (include/tnqvm.h): argument marshalling only.

Every step of the contraction path runs inside libtnqvm's sm_100a kernels; this module
converts numpy / torch arguments to the C-ABI and back.  There is no CPU fallback: a
missing or unloadable library raises, and device calls without a B200 raise TnqvmError.
"""
from __future__ import annotations

import ctypes as C
import json
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libtnqvm.so")

OK, EINVAL, ENOTUNITARY, ENOTCPTP, EINFEASIBLE, ENOMEM, ECUDA, ENCCL, ESTATE = 0, -1, -2, -3, -4, -5, -6, -7, -8
C64, C128 = 0, 1

EXPORTED = [
    "tnqvm_version", "tnqvm_last_error", "tnqvm_plan_opts_default",
    "tnqvm_circuit_create", "tnqvm_circuit_destroy", "tnqvm_apply_gate", "tnqvm_apply_kraus",
    "tnqvm_plan_create", "tnqvm_plan_json", "tnqvm_plan_get_info", "tnqvm_plan_destroy",
    "tnqvm_ctx_create", "tnqvm_ctx_destroy", "tnqvm_nccl_unique_id", "tnqvm_ctx_last_stats",
    "tnqvm_ctx_set_timing", "tnqvm_amplitude", "tnqvm_amplitude_batch", "tnqvm_amplitudes", "tnqvm_expectation",
    "tnqvm_eval_slices", "tnqvm_permute_device", "tnqvm_gemm_device", "tnqvm_gemm_gather_device",
    "tnqvm_plan_autotune", "tnqvm_plan_raw_network",
    "tnqvm_network_export", "tnqvm_plan_rank_slices", "tnqvm_ctx_class_stats", "tnqvm_ctx_set_roofline",
    "tnqvm_ctx_group_slots", "tnqvm_plan_kernel_classes", "tnqvm_expectation_wfslice", "tnqvm_sample",
    "tnqvm_plan_program_json",
]
# kernel classes of tnqvm_ctx_class_stats (include/tnqvm.h)
KERNEL_CLASSES = ["small", "strided", "skinny", "gemm_tc", "gemm_dmma", "gemm_simt", "splitk", "permute", "accum"]


class TnqvmError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"tnqvm error {code}: {msg}")
        self.code = code


class c128(C.Structure):
    _fields_ = [("re", C.c_double), ("im", C.c_double)]


class PauliTerm(C.Structure):
    _fields_ = [("coeff", C.c_double), ("nops", C.c_int32), ("qubits", C.POINTER(C.c_int32)),
                ("paulis", C.c_char_p)]


class PlanOpts(C.Structure):
    _fields_ = [("seed", C.c_uint64), ("restarts", C.c_int32), ("threads", C.c_int32),
                ("time_cap_s", C.c_double), ("dtype", C.c_int32), ("cancel_conjugates", C.c_int32),
                ("min_slices", C.c_uint64), ("cost_model", C.c_int32), ("partition", C.c_int32)]


class PlanInfo(C.Structure):
    _fields_ = [("n_leaves", C.c_int32), ("n_steps", C.c_int32), ("n_wires", C.c_int32),
                ("n_open", C.c_int32), ("n_sliced", C.c_int32), ("n_slices", C.c_uint64),
                ("log2_macs_unsliced", C.c_double), ("log2_macs_sliced", C.c_double),
                ("log2_max_intermediate", C.c_double), ("flops_sliced", C.c_double),
                ("bytes_sliced", C.c_double), ("noisy", C.c_int32), ("dtype", C.c_int32)]


class ClassStats(C.Structure):
    _fields_ = [("ms", C.c_double), ("bytes", C.c_double), ("flops", C.c_double), ("launches", C.c_int64),
                ("roof_ms", C.c_double), ("roof_hbm_ms", C.c_double)]


class Stats(C.Structure):
    _fields_ = [("ms_total", C.c_double), ("ms_gemm", C.c_double), ("gemm_launches", C.c_int64),
                ("kernel_launches", C.c_int64), ("gemm_bytes", C.c_double), ("gemm_flops", C.c_double),
                ("flops", C.c_double), ("bytes", C.c_double), ("h2d_bytes", C.c_uint64),
                ("d2h_bytes", C.c_uint64), ("host_ms", C.c_double), ("graph", C.c_int32), ("pad_", C.c_int32)]


ALLOC_FN = C.CFUNCTYPE(C.c_void_p, C.c_size_t, C.c_void_p)
FREE_FN = C.CFUNCTYPE(None, C.c_void_p, C.c_void_p)

_lib = None


def lib():
    """Load libtnqvm.so (built in-tree); raise if absent -- there is no fallback."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} not built; run __graft_entry__.build()")
    L = C.CDLL(LIB_PATH)
    P = C.POINTER
    L.tnqvm_version.restype = C.c_int
    L.tnqvm_last_error.restype = C.c_char_p
    L.tnqvm_plan_opts_default.argtypes = [P(PlanOpts)]
    L.tnqvm_circuit_create.argtypes = [C.c_int32, P(C.c_void_p)]
    L.tnqvm_circuit_destroy.argtypes = [C.c_void_p]
    L.tnqvm_apply_gate.argtypes = [C.c_void_p, P(c128), P(C.c_int32), C.c_int32]
    L.tnqvm_apply_kraus.argtypes = [C.c_void_p, P(c128), C.c_int32, P(C.c_int32), C.c_int32]
    L.tnqvm_plan_create.argtypes = [C.c_void_p, P(C.c_int32), C.c_int32, C.c_uint64, P(PlanOpts), P(C.c_void_p)]
    L.tnqvm_plan_json.argtypes = [C.c_void_p, C.c_char_p, C.c_size_t, P(C.c_size_t)]
    L.tnqvm_plan_get_info.argtypes = [C.c_void_p, P(PlanInfo)]
    L.tnqvm_plan_destroy.argtypes = [C.c_void_p]
    L.tnqvm_network_export.argtypes = [C.c_void_p, P(C.c_int8), C.c_char_p, C.c_size_t, P(C.c_size_t)]
    L.tnqvm_plan_rank_slices.argtypes = [C.c_void_p, C.c_int, C.c_int, P(C.c_uint64), C.c_uint64, P(C.c_uint64)]
    L.tnqvm_plan_raw_network.argtypes = [P(C.c_int32), P(C.c_int32), C.c_int32, P(C.c_int32), C.c_int32,
                                         C.c_uint64, P(PlanOpts), C.c_char_p, C.c_size_t, P(C.c_size_t)]
    L.tnqvm_ctx_create.argtypes = [C.c_int, C.c_int, C.c_int, C.c_void_p, C.c_void_p, ALLOC_FN, FREE_FN,
                                   C.c_void_p, P(C.c_void_p)]
    L.tnqvm_ctx_destroy.argtypes = [C.c_void_p]
    L.tnqvm_nccl_unique_id.argtypes = [C.c_void_p]
    L.tnqvm_ctx_last_stats.argtypes = [C.c_void_p, P(Stats)]
    L.tnqvm_ctx_set_timing.argtypes = [C.c_void_p, C.c_int]
    L.tnqvm_ctx_class_stats.argtypes = [C.c_void_p, C.c_int, P(ClassStats)]
    L.tnqvm_ctx_set_roofline.argtypes = [C.c_void_p, C.c_double, C.c_double, C.c_double]
    L.tnqvm_expectation_wfslice.argtypes = [C.c_void_p, C.c_void_p, P(PauliTerm), C.c_int32, C.c_int32, C.c_uint64,
                                            P(PlanOpts), P(c128), P(c128)]
    L.tnqvm_sample.argtypes = [C.c_void_p, C.c_void_p, P(C.c_double), C.c_int32, C.c_int32, C.c_uint64, P(PlanOpts),
                               P(C.c_int8), P(C.c_double)]
    L.tnqvm_plan_program_json.argtypes = [C.c_void_p, C.c_char_p, C.c_size_t, P(C.c_size_t)]
    L.tnqvm_plan_kernel_classes.argtypes = [C.c_void_p, P(C.c_int64)]
    L.tnqvm_ctx_group_slots.argtypes = [C.c_void_p, P(c128), C.c_int64, P(C.c_int64)]
    L.tnqvm_amplitude.argtypes = [C.c_void_p, C.c_void_p, P(C.c_int8), P(c128)]
    L.tnqvm_amplitude_batch.argtypes = [C.c_void_p, C.c_void_p, P(C.c_int8), C.c_int32, P(c128)]
    L.tnqvm_amplitudes.argtypes = [C.c_void_p, C.c_void_p, P(C.c_int8), P(c128)]
    L.tnqvm_expectation.argtypes = [C.c_void_p, C.c_void_p, P(PauliTerm), C.c_int32, C.c_uint64, P(PlanOpts),
                                    P(c128), P(c128)]
    L.tnqvm_eval_slices.argtypes = [C.c_void_p, C.c_void_p, P(C.c_int8), P(C.c_uint64), C.c_int32, P(c128)]
    L.tnqvm_permute_device.argtypes = [C.c_void_p, C.c_int, C.c_void_p, C.c_void_p, C.c_int32, P(C.c_int32)]
    L.tnqvm_plan_autotune.argtypes = [C.c_void_p, C.c_void_p, C.c_uint64, C.c_void_p, P(C.c_uint64), C.c_int32,
                                      P(C.c_int8), C.c_int32, C.c_int32, P(C.c_void_p), P(C.c_double)]
    L.tnqvm_gemm_gather_device.argtypes = [C.c_void_p, C.c_int, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int32,
                                           C.c_int32, C.c_int32, P(C.c_int64), P(C.c_int64)]
    L.tnqvm_gemm_device.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_void_p, C.c_void_p, C.c_void_p,
                                    C.c_int64, C.c_int64, C.c_int64]
    _lib = L
    return L


def _check(code):
    if code != 0:
        raise TnqvmError(code, lib().tnqvm_last_error().decode(errors="replace"))


def _c128_array(M):
    M = np.ascontiguousarray(np.asarray(M, dtype=np.complex128))
    arr = (c128 * M.size)()
    flat = M.reshape(-1)
    for i, z in enumerate(flat):
        arr[i].re = z.real
        arr[i].im = z.imag
    return arr


def _i32(xs):
    xs = list(int(x) for x in xs)
    return (C.c_int32 * max(1, len(xs)))(*xs)


def _i64(xs):
    xs = list(int(x) for x in xs)
    return (C.c_int64 * max(1, len(xs)))(*xs)


def _to_np(arr, n):
    return np.array([complex(arr[i].re, arr[i].im) for i in range(n)], dtype=np.complex128)


def plan_opts(seed=0, restarts=64, threads=0, time_cap_s=0.0, dtype=C64, cancel_conjugates=1, min_slices=1,
              cost_model=1, partition=1):
    o = PlanOpts()
    lib().tnqvm_plan_opts_default(C.byref(o))
    o.seed, o.restarts, o.threads, o.time_cap_s = seed, restarts, threads, time_cap_s
    o.dtype, o.cancel_conjugates, o.min_slices, o.cost_model = dtype, cancel_conjugates, min_slices, cost_model
    o.partition = partition
    return o


class Circuit:
    """tnqvm_circuit: an ordered list of gates and Kraus channels (host only)."""

    def __init__(self, nq):
        self.nq = nq
        h = C.c_void_p()
        _check(lib().tnqvm_circuit_create(nq, C.byref(h)))
        self.h = h

    @classmethod
    def from_oplist(cls, oplist):
        c = cls(oplist.nq)
        for op in oplist.ops:
            if op.kind == "gate":
                c.apply_gate(op.mats[0], op.qubits)
            else:
                c.apply_kraus(op.mats, op.qubits)
        return c

    def apply_gate(self, U, qubits):
        _check(lib().tnqvm_apply_gate(self.h, _c128_array(U), _i32(qubits), len(qubits)))

    def apply_kraus(self, Ks, qubits):
        Ks = np.stack([np.asarray(K, dtype=np.complex128) for K in Ks])
        _check(lib().tnqvm_apply_kraus(self.h, _c128_array(Ks), len(Ks), _i32(qubits), len(qubits)))

    def __del__(self):
        if getattr(self, "h", None) and _lib is not None:
            _lib.tnqvm_circuit_destroy(self.h)
            self.h = None


class Plan:
    """tnqvm_plan: network + contraction path + slicing (host only; no GPU needed)."""

    def __init__(self, circuit: Circuit, out_qubits=(), max_slice_bytes=1 << 34, **opts):
        self.circuit = circuit
        self.out_qubits = list(out_qubits)
        h = C.c_void_p()
        o = plan_opts(**opts)
        _check(lib().tnqvm_plan_create(circuit.h, _i32(self.out_qubits), len(self.out_qubits),
                                       int(max_slice_bytes), C.byref(o), C.byref(h)))
        self.h = h

    @classmethod
    def _adopt(cls, circuit: Circuit, handle, out_qubits=()):
        """Wrap a plan handle created by the library (tnqvm_plan_autotune)."""
        p = cls.__new__(cls)
        p.circuit = circuit
        p.out_qubits = list(out_qubits)
        p.h = handle
        return p

    def json(self) -> str:
        n = C.c_size_t()
        _check(lib().tnqvm_plan_json(self.h, None, 0, C.byref(n)))
        buf = C.create_string_buffer(n.value + 1)
        _check(lib().tnqvm_plan_json(self.h, buf, n.value + 1, C.byref(n)))
        return buf.value.decode()

    def dict(self):
        return json.loads(self.json())

    def info(self) -> dict:
        i = PlanInfo()
        _check(lib().tnqvm_plan_get_info(self.h, C.byref(i)))
        return {f: getattr(i, f) for f, _ in PlanInfo._fields_}

    def network(self, bits=None) -> dict:
        """The network handed to the planner (builder output) with leaf values."""
        b = (C.c_int8 * len(bits))(*[int(x) for x in bits]) if bits is not None else None
        n = C.c_size_t()
        _check(lib().tnqvm_network_export(self.h, b, None, 0, C.byref(n)))
        buf = C.create_string_buffer(n.value + 1)
        _check(lib().tnqvm_network_export(self.h, b, buf, n.value + 1, C.byref(n)))
        d = json.loads(buf.value.decode())
        for lf in d["leaves"]:
            v = np.array(lf["data"], dtype=np.float64)
            lf["data"] = (v[0::2] + 1j * v[1::2]).reshape((2,) * len(lf["wires"]))
        d["scalar"] = complex(*d["scalar"])
        return d

    def program(self) -> dict:
        """The compiled launch list (host only): ops, tensor layouts, arena sizes."""
        n = C.c_size_t()
        _check(lib().tnqvm_plan_program_json(self.h, None, 0, C.byref(n)))
        buf = C.create_string_buffer(n.value + 1)
        _check(lib().tnqvm_plan_program_json(self.h, buf, n.value + 1, C.byref(n)))
        return json.loads(buf.value.decode())

    def kernel_classes(self) -> dict:
        """Ops per kernel class of the compiled launch list (host only)."""
        counts = (C.c_int64 * len(KERNEL_CLASSES))()
        _check(lib().tnqvm_plan_kernel_classes(self.h, counts))
        return {n: int(counts[i]) for i, n in enumerate(KERNEL_CLASSES)}

    def rank_slices(self, rank, world):
        n = C.c_uint64()
        _check(lib().tnqvm_plan_rank_slices(self.h, rank, world, None, 0, C.byref(n)))
        out = (C.c_uint64 * max(1, n.value))()
        _check(lib().tnqvm_plan_rank_slices(self.h, rank, world, out, n.value, C.byref(n)))
        return [int(out[i]) for i in range(n.value)]

    def sliced_wires(self):
        d = self.dict()
        wires = {w["id"]: w for w in d["wires"]}
        return [wires[i] for i in d["sliced"]]

    def __del__(self):
        if getattr(self, "h", None) and _lib is not None:
            _lib.tnqvm_plan_destroy(self.h)
            self.h = None


class Context:
    """tnqvm_ctx: device, rank/world, CUDA stream, optional NCCL communicator (world > 1
    without ``nccl_id``: an emulated rank that evaluates only its own slice groups).  Device
    memory comes from the torch caching allocator when ``use_torch_allocator``."""

    def __init__(self, device=0, rank=0, world=1, nccl_id: bytes | None = None, stream=None,
                 use_torch_allocator=True):
        self._keep = []
        alloc = ALLOC_FN()
        free = FREE_FN()
        if use_torch_allocator:
            import torch
            dev = device
            talloc, tdelete = torch.cuda.caching_allocator_alloc, torch.cuda.caching_allocator_delete
            if stream is None:  # stream-order with torch's current stream on this device
                stream = torch.cuda.current_stream(device).cuda_stream

            def _alloc(n, ud):
                try:
                    return talloc(int(n), dev, stream if stream else None)
                except Exception:  # noqa: BLE001 -- reported as ENOMEM by the library
                    return None

            def _free(p, ud):
                try:
                    tdelete(p)
                except Exception:  # noqa: BLE001 -- interpreter shutdown
                    pass

            alloc, free = ALLOC_FN(_alloc), FREE_FN(_free)
            self._keep += [alloc, free]
        idbuf = None
        if nccl_id is not None:
            idbuf = C.create_string_buffer(bytes(nccl_id), 128)
            self._keep.append(idbuf)
        h = C.c_void_p()
        _check(lib().tnqvm_ctx_create(device, rank, world, C.cast(idbuf, C.c_void_p) if idbuf else None,
                                      C.c_void_p(stream) if stream else None, alloc, free, None, C.byref(h)))
        self.h = h
        self.device, self.rank, self.world = device, rank, world

    def set_timing(self, on=True):
        _check(lib().tnqvm_ctx_set_timing(self.h, 1 if on else 0))

    def set_roofline(self, hbm_gbs, c64_tflops, c128_tflops):
        _check(lib().tnqvm_ctx_set_roofline(self.h, hbm_gbs, c64_tflops, c128_tflops))

    def class_stats(self) -> dict:
        """Per-kernel-class device time / algorithmic bytes / flops / ops of the last call
        made with set_timing(True)."""
        out = {}
        for i, name in enumerate(KERNEL_CLASSES):
            s = ClassStats()
            _check(lib().tnqvm_ctx_class_stats(self.h, i, C.byref(s)))
            out[name] = {f: getattr(s, f) for f, _ in ClassStats._fields_}
        return out

    def group_slots(self) -> np.ndarray:
        """The 8 x 2^k complex128 group slots of the last amplitude(s) call (after the
        cross-rank reduction; an emulated rank's own groups only)."""
        n = C.c_int64()
        _check(lib().tnqvm_ctx_group_slots(self.h, None, 0, C.byref(n)))
        out = (c128 * max(1, n.value))()
        _check(lib().tnqvm_ctx_group_slots(self.h, out, n.value, C.byref(n)))
        return _to_np(out, n.value).reshape(8, -1)

    def stats(self) -> dict:
        s = Stats()
        _check(lib().tnqvm_ctx_last_stats(self.h, C.byref(s)))
        return {f: getattr(s, f) for f, _ in Stats._fields_}

    def amplitude(self, plan: Plan, bits) -> complex:
        b = (C.c_int8 * len(bits))(*[int(x) for x in bits])
        out = c128()
        _check(lib().tnqvm_amplitude(self.h, plan.h, b, C.byref(out)))
        return complex(out.re, out.im)

    def amplitude_batch(self, plan: Plan, bits_rows) -> np.ndarray:
        """Amplitudes of many bitstrings (rows) of one plan: tnqvm_amplitude_batch."""
        rows = [[int(x) for x in r] for r in bits_rows]
        nb = len(rows)
        flat = [x for r in rows for x in r]
        b = (C.c_int8 * max(1, len(flat)))(*flat)
        out = (c128 * max(1, nb))()
        _check(lib().tnqvm_amplitude_batch(self.h, plan.h, b, nb, out))
        return _to_np(out, nb)

    def autotune_plan(self, circuit: Circuit, max_slice_bytes, seeds, bits_rows, reps=3, **opts):
        """tnqvm_plan_autotune: the fastest measured plan among the seeds' plans; returns
        (Plan, [ms per seed])."""
        rows = [[int(x) for x in r] for r in bits_rows]
        flat = [x for r in rows for x in r]
        b = (C.c_int8 * max(1, len(flat)))(*flat)
        sd = (C.c_uint64 * len(seeds))(*[int(x) for x in seeds])
        ms = (C.c_double * len(seeds))()
        h = C.c_void_p()
        o = plan_opts(**opts)
        _check(lib().tnqvm_plan_autotune(self.h, circuit.h, int(max_slice_bytes), C.byref(o), sd, len(seeds), b,
                                         len(rows), int(reps), C.byref(h), ms))
        return Plan._adopt(circuit, h), [ms[i] for i in range(len(seeds))]

    def amplitudes(self, plan: Plan, bits) -> np.ndarray:
        b = (C.c_int8 * len(bits))(*[int(x) for x in bits])
        k = sum(1 for x in bits if int(x) < 0)
        n = plan.info()["n_open"]
        out = (c128 * (1 << n))()
        _check(lib().tnqvm_amplitudes(self.h, plan.h, b, out))
        v = _to_np(out, 1 << n)
        if n != k:  # noisy: 2^k x 2^k block
            v = v.reshape(1 << k, 1 << k)
        return v

    def eval_slices(self, plan: Plan, bits, slice_ids) -> np.ndarray:
        b = (C.c_int8 * len(bits))(*[int(x) for x in bits])
        ids = (C.c_uint64 * len(slice_ids))(*[int(s) for s in slice_ids])
        n = plan.info()["n_open"]
        rl = 1 << n
        out = (c128 * (rl * len(slice_ids)))()
        _check(lib().tnqvm_eval_slices(self.h, plan.h, b, ids, len(slice_ids), out))
        return _to_np(out, rl * len(slice_ids)).reshape(len(slice_ids), rl)

    @staticmethod
    def _terms(terms):
        arr = (PauliTerm * max(1, len(terms)))()
        keep = []
        for i, (c, t) in enumerate(terms):
            qs = _i32([q for q, _ in t])
            ps = C.c_char_p("".join(p for _, p in t).encode())
            keep += [qs, ps]
            arr[i].coeff = float(c)
            arr[i].nops = len(t)
            arr[i].qubits = C.cast(qs, C.POINTER(C.c_int32))
            arr[i].paulis = ps
        return arr, keep

    def expectation(self, circuit: Circuit, terms, max_slice_bytes=1 << 34, per_term=False, **opts):
        """terms = [(coeff, [(q, 'X'|'Y'|'Z'|'I'|'0'|'1'), ...]), ...] (bra-ket network)"""
        arr, keep = self._terms(terms)
        tot = c128()
        per = (c128 * max(1, len(terms)))()
        o = plan_opts(**opts)
        _check(lib().tnqvm_expectation(self.h, circuit.h, arr, len(terms), int(max_slice_bytes), C.byref(o),
                                       C.byref(tot), per))
        total = complex(tot.re, tot.im)
        if per_term:
            return total, _to_np(per, len(terms))
        return total

    def expectation_wfslice(self, circuit: Circuit, terms, rank_max, max_slice_bytes=1 << 34, per_term=False,
                            **opts):
        """Expectation value by wave-function slicing (tnqvm_expectation_wfslice)."""
        arr, keep = self._terms(terms)
        tot = c128()
        per = (c128 * max(1, len(terms)))()
        o = plan_opts(**opts)
        _check(lib().tnqvm_expectation_wfslice(self.h, circuit.h, arr, len(terms), int(rank_max), int(max_slice_bytes),
                                               C.byref(o), C.byref(tot), per))
        total = complex(tot.re, tot.im)
        if per_term:
            return total, _to_np(per, len(terms))
        return total

    def sample(self, circuit: Circuit, uniforms, block=1, max_slice_bytes=1 << 34, **opts):
        """Bit-string samples (tnqvm_sample): (bits [nshots x nq] int8, probabilities [nshots])."""
        us = [float(u) for u in uniforms]
        n = len(us)
        nq = circuit.nq
        ua = (C.c_double * max(1, n))(*us)
        bits = (C.c_int8 * max(1, n * nq))()
        probs = (C.c_double * max(1, n))()
        o = plan_opts(**opts)
        _check(lib().tnqvm_sample(self.h, circuit.h, ua, n, int(block), int(max_slice_bytes), C.byref(o), bits, probs))
        return (np.ctypeslib.as_array(bits)[:n * nq].reshape(n, nq).copy(),
                np.ctypeslib.as_array(probs)[:n].copy())

    def permute(self, dtype, src_ptr, dst_ptr, rank, perm):
        _check(lib().tnqvm_permute_device(self.h, dtype, C.c_void_p(src_ptr), C.c_void_p(dst_ptr), rank, _i32(perm)))

    def gemm(self, dtype, method, X_ptr, Y_ptr, C_ptr, N, K, M):
        _check(lib().tnqvm_gemm_device(self.h, dtype, method, C.c_void_p(X_ptr), C.c_void_p(Y_ptr),
                                       C.c_void_p(C_ptr), N, K, M))

    def gemm_gather(self, dtype, X_ptr, Y_ptr, C_ptr, nn, nk, nm, sxn, sxk):
        """C = X Y with X element (n, k) at sum_i bit_i(n) sxn[i] + sum_i bit_i(k) sxk[i]."""
        _check(lib().tnqvm_gemm_gather_device(self.h, dtype, C.c_void_p(X_ptr), C.c_void_p(Y_ptr), C.c_void_p(C_ptr),
                                              nn, nk, nm, _i64(sxn), _i64(sxk)))

    def close(self):
        if getattr(self, "h", None):
            lib().tnqvm_ctx_destroy(self.h)
            self.h = None

    def __del__(self):
        if _lib is not None:
            self.close()


def plan_raw_network(leaves, open_wires=(), budget_elems=1 << 62, **opts) -> dict:
    """Planner test hook: leaves = [[wire ids], ...] (binary wires)."""
    ranks = _i32([len(l) for l in leaves])
    wires = _i32([w for l in leaves for w in l])
    op = _i32(open_wires)
    o = plan_opts(**opts)
    n = C.c_size_t()
    _check(lib().tnqvm_plan_raw_network(ranks, wires, len(leaves), op, len(open_wires), int(budget_elems),
                                        C.byref(o), None, 0, C.byref(n)))
    buf = C.create_string_buffer(n.value + 1)
    _check(lib().tnqvm_plan_raw_network(ranks, wires, len(leaves), op, len(open_wires), int(budget_elems),
                                        C.byref(o), buf, n.value + 1, C.byref(n)))
    return json.loads(buf.value.decode())


def nccl_unique_id() -> bytes:
    buf = C.create_string_buffer(128)
    _check(lib().tnqvm_nccl_unique_id(buf))
    return buf.raw
