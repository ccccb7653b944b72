"""ctypes binding of libsymel_cuda.so (include/symel_cuda.h), shaped like the reference's
EnergySystem + Assembler pair (registry.hpp:111-445, assembly.hpp:90-187):

    asm = DeviceAssembler()
    x = asm.add_array("x", n, 3, is_dof=True); asm.set_array(x, pos)
    t = asm.add_connectivity("tets", 4);       asm.set_elements(t, conn)
    e = asm.add_energy("elastic", t, tape_bytes, inputs, dof_slots)
    E = asm.assemble()                          # raises SymelError like symel::Error
    g, H = asm.gradient(), asm.hessian()

There is no CPU path here: creating a DeviceAssembler without a GPU raises.
"""
from __future__ import annotations

import ctypes as C
import dataclasses
import os
from typing import Optional, Sequence

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libsymel_cuda.so")

OK, E_ARG, E_CUDA, E_COMPILE, E_NONFINITE, E_STATE, E_TAPE, E_NODEVICE = range(8)
IN_ITEM, IN_ELEM, IN_PARAM, IN_SUM = range(4)
ASM_DETERMINISTIC, ASM_ATOMIC, ASM_ORDERED = 0, 1, 2
ENERGY_SPD = 1
ENERGY_EXACT = 2

MODES = {"deterministic": ASM_DETERMINISTIC, "atomic": ASM_ATOMIC, "ordered": ASM_ORDERED}


class SymelError(RuntimeError):
    """Mirrors symel::Error (expr.hpp:21-24); `code` is the C-ABI status."""

    def __init__(self, code: int, msg: str):
        super().__init__(msg)
        self.code = code


class InputSrc(C.Structure):
    _fields_ = [("kind", C.c_uint32), ("array", C.c_uint32), ("tuple_slot", C.c_uint32), ("comp", C.c_uint32)]


class Status(C.Structure):
    _fields_ = [("code", C.c_int32), ("energy", C.c_int32), ("element", C.c_int64)]


class Timings(C.Structure):
    _fields_ = [("eval_ms", C.c_double), ("assemble_ms", C.c_double), ("pattern_ms", C.c_double),
                ("compile_ms", C.c_double)]


EXPORTS = [
    "symel_cuda_abi_version", "symel_cuda_create", "symel_cuda_destroy", "symel_cuda_last_error",
    "symel_cuda_set_cache_dir", "symel_cuda_add_array", "symel_cuda_set_array", "symel_cuda_get_array",
    "symel_cuda_array_device_ptr", "symel_cuda_add_connectivity", "symel_cuda_set_elements",
    "symel_cuda_add_energy", "symel_cuda_set_param", "symel_cuda_set_energy_flags", "symel_cuda_set_pins",
    "symel_cuda_assemble", "symel_cuda_energy_only", "symel_cuda_guard_min", "symel_cuda_pattern_info",
    "symel_cuda_copy_pattern", "symel_cuda_copy_gradient", "symel_cuda_copy_hessian",
    "symel_cuda_device_results", "symel_cuda_active_count", "symel_cuda_copy_active", "symel_cuda_energy_parts",
    "symel_cuda_matvec", "symel_cuda_block_jacobi", "symel_cuda_pcg", "symel_cuda_gather_dofs",
    "symel_cuda_scatter_dofs",
    "symel_cuda_element_outputs", "symel_cuda_get_timings", "symel_cuda_kernel_source",
    "symel_cuda_launch_count", "symel_cuda_fp64_peak", "symel_cuda_precompile", "symel_cuda_sync",
    "symel_cuda_stream", "symel_cuda_energy_info", "symel_cuda_plan_info", "symel_cuda_cache_stats",
]


class EnergyStats(C.Structure):
    _fields_ = [("tape_ops", C.c_uint64), ("fast_ops", C.c_uint64), ("frontier", C.c_uint32),
                ("n_dofs", C.c_uint32), ("n_inputs", C.c_uint32), ("n_outputs", C.c_uint32),
                ("n_items", C.c_uint32), ("flags", C.c_uint32)]

_lib = None


def load_library(path: str = LIB_PATH) -> C.CDLL:
    """Loads the C-ABI library; raises if it has not been built (no silent fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise ImportError(f"{path} missing: run __graft_entry__.build() (the CUDA path is the only path)")
    lib = C.CDLL(path)
    P, I, U64, D = C.c_void_p, C.c_int, C.c_uint64, C.c_double
    sig = {
        "symel_cuda_abi_version": ([], I),
        "symel_cuda_create": ([I, C.POINTER(P)], I),
        "symel_cuda_destroy": ([P], None),
        "symel_cuda_last_error": ([P], C.c_char_p),
        "symel_cuda_set_cache_dir": ([P, C.c_char_p], I),
        "symel_cuda_cache_stats": ([P, P], I),
        "symel_cuda_add_array": ([P, C.c_char_p, U64, C.c_uint32, I, C.POINTER(I)], I),
        "symel_cuda_set_array": ([P, I, P, U64], I),
        "symel_cuda_get_array": ([P, I, P, U64], I),
        "symel_cuda_array_device_ptr": ([P, I, C.POINTER(P)], I),
        "symel_cuda_add_connectivity": ([P, C.c_char_p, C.c_uint32, C.POINTER(I)], I),
        "symel_cuda_set_elements": ([P, I, P, U64], I),
        "symel_cuda_add_energy": ([P, C.c_char_p, I, P, U64, P, C.c_uint32, P, C.c_uint32, P, C.c_uint32,
                                   C.c_uint32, P, U64, I, P, U64, C.POINTER(I)], I),
        "symel_cuda_set_param": ([P, I, C.c_uint32, D], I),
        "symel_cuda_set_energy_flags": ([P, I, C.c_uint32], I),
        "symel_cuda_set_pins": ([P, P, U64], I),
        "symel_cuda_assemble": ([P, C.c_uint32, C.POINTER(D), C.POINTER(Status)], I),
        "symel_cuda_energy_only": ([P, C.POINTER(D)], I),
        "symel_cuda_guard_min": ([P, C.POINTER(D)], I),
        "symel_cuda_pattern_info": ([P, C.POINTER(I), C.POINTER(U64), C.POINTER(U64), C.POINTER(U64)], I),
        "symel_cuda_copy_pattern": ([P, P, P], I),
        "symel_cuda_copy_gradient": ([P, P], I),
        "symel_cuda_copy_hessian": ([P, P], I),
        "symel_cuda_device_results": ([P, P, P, P, P], I),
        "symel_cuda_active_count": ([P, I, C.POINTER(U64)], I),
        "symel_cuda_energy_parts": ([P, C.POINTER(C.c_double), C.c_uint32], I),
        "symel_cuda_matvec": ([P, C.c_void_p, C.c_void_p, C.c_uint32], I),
        "symel_cuda_gather_dofs": ([P, C.c_void_p, C.c_uint32], I),
        "symel_cuda_scatter_dofs": ([P, C.c_void_p, C.c_uint32], I),
        "symel_cuda_block_jacobi": ([P, C.c_double, C.c_void_p, C.c_uint32], I),
        "symel_cuda_pcg": ([P, C.c_double, C.c_void_p, C.c_void_p, C.c_double, C.c_int32, C.c_uint32,
                            C.POINTER(PcgResult)], I),
        "symel_cuda_copy_active": ([P, I, P], I),
        "symel_cuda_element_outputs": ([P, I, U64, U64, C.c_uint32, P], I),
        "symel_cuda_get_timings": ([P, C.POINTER(Timings)], I),
        "symel_cuda_kernel_source": ([P, I, C.c_uint32, P, U64, C.POINTER(U64)], I),
        "symel_cuda_launch_count": ([P, C.POINTER(U64)], I),
        "symel_cuda_fp64_peak": ([P, C.POINTER(D)], I),
        "symel_cuda_precompile": ([P, I, C.c_uint32], I),
        "symel_cuda_energy_info": ([P, I, C.POINTER(EnergyStats)], I),
        "symel_cuda_plan_info": ([P, P], I),
        "symel_cuda_sync": ([P], I),
        "symel_cuda_stream": ([P, C.POINTER(P)], I),
    }
    for name, (args, res) in sig.items():
        f = getattr(lib, name)
        f.argtypes = args
        f.restype = res
    _lib = lib
    return lib


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(C.c_void_p)


@dataclasses.dataclass
class Bcrs:
    """BcrsMatrix (assembly.hpp:18-75)."""
    b: int
    row_ptr: np.ndarray
    col_idx: np.ndarray
    values: np.ndarray

    @property
    def n_block_rows(self) -> int:
        return self.row_ptr.size - 1

    def find_block(self, r: int, c: int) -> int:
        lo, hi = self.row_ptr[r], self.row_ptr[r + 1]
        k = lo + np.searchsorted(self.col_idx[lo:hi], c)
        return int(k) if k < hi and self.col_idx[k] == c else -1

    def dump(self) -> str:
        """BcrsMatrix::dump (assembly.hpp:60-74): "b n_block_rows n_blocks", then one line per
        stored block in row order, "(r c)" and the b*b values row-major as %.17g."""
        b = int(self.b)
        out = ["%d %d %d\n" % (b, self.n_block_rows, self.col_idx.size)]
        v = self.values.reshape(-1, b * b)
        for r in range(self.n_block_rows):
            for k in range(int(self.row_ptr[r]), int(self.row_ptr[r + 1])):
                out.append("(%d %d)" % (r, int(self.col_idx[k])) + "".join(" %.17g" % x for x in v[k]) + "\n")
        return "".join(out)

    def to_dense(self) -> np.ndarray:
        b, n = self.b, self.n_block_rows
        D = np.zeros((n * b, n * b))
        v = self.values.reshape(-1, b, b)
        for r in range(n):
            for k in range(self.row_ptr[r], self.row_ptr[r + 1]):
                c = self.col_idx[k]
                D[r * b:(r + 1) * b, c * b:(c + 1) * b] = v[k]
        return D


class PcgResult(C.Structure):
    """symel_cuda_pcg_result (PcgResult, optimizer.hpp:24-29, + device solve time)."""
    _fields_ = [("iters", C.c_int32), ("converged", C.c_int32), ("neg_curvature", C.c_int32),
                ("reserved", C.c_int32), ("rel_residual", C.c_double), ("solve_ms", C.c_double)]


PTR_DEVICE = 1


class DeviceAssembler:
    def __init__(self, device: int = 0, cache_dir: Optional[str] = None):
        self.lib = load_library()
        h = C.c_void_p()
        rc = self.lib.symel_cuda_create(device, C.byref(h))
        if rc != OK:
            raise SymelError(rc, "symel_cuda_create failed: " + self.lib.symel_cuda_last_error(None).decode())
        self.h = h
        self.device = device
        self._keep = []
        if cache_dir is None:
            cache_dir = os.environ.get("SYMEL_CUDA_CACHE", os.path.join(_HERE, "_cache"))
        self._check(self.lib.symel_cuda_set_cache_dir(self.h, cache_dir.encode()))
        self.energy_names = []

    def close(self):
        if getattr(self, "h", None):
            self.lib.symel_cuda_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _check(self, rc: int):
        if rc != OK:
            raise SymelError(rc, self.lib.symel_cuda_last_error(self.h).decode())

    # ---- system
    def add_array(self, name: str, items: int, comps: int, is_dof: bool = False) -> int:
        i = C.c_int()
        self._check(self.lib.symel_cuda_add_array(self.h, name.encode(), items, comps, int(is_dof), C.byref(i)))
        return i.value

    def set_array(self, aid: int, data: np.ndarray) -> None:
        if self.device < 0:
            return  # codegen-only context: shapes matter, values do not
        d = np.ascontiguousarray(data, dtype=np.float64).ravel()
        self._check(self.lib.symel_cuda_set_array(self.h, aid, _ptr(d), d.size))

    def get_array(self, aid: int, count: int) -> np.ndarray:
        out = np.empty(count)
        self._check(self.lib.symel_cuda_get_array(self.h, aid, _ptr(out), count))
        return out

    def array_device_ptr(self, aid: int) -> int:
        p = C.c_void_p()
        self._check(self.lib.symel_cuda_array_device_ptr(self.h, aid, C.byref(p)))
        return p.value

    def add_connectivity(self, name: str, arity: int) -> int:
        i = C.c_int()
        self._check(self.lib.symel_cuda_add_connectivity(self.h, name.encode(), arity, C.byref(i)))
        return i.value

    def set_elements(self, cid: int, conn: np.ndarray) -> None:
        c = np.ascontiguousarray(conn, dtype=np.int64)
        n = c.shape[0] if c.ndim == 2 else c.size
        self._check(self.lib.symel_cuda_set_elements(self.h, cid, _ptr(c), n))

    def add_energy(self, name: str, conn: int, tape: bytes, inputs: Sequence, dof_slots: Sequence[int],
                   sum_items: Optional[np.ndarray] = None, act_tape: Optional[bytes] = None, act_kind: int = 0,
                   guard_tape: Optional[bytes] = None, params: Optional[dict] = None, flags: int = 0) -> int:
        ins = (InputSrc * len(inputs))(*[InputSrc(*x) for x in inputs])
        ds = np.ascontiguousarray(dof_slots, dtype=np.uint32)
        if sum_items is not None:
            si = np.ascontiguousarray(sum_items, dtype=np.float64)
            n_items, arity = si.shape
            sp = _ptr(si)
            self._keep.append(si)
        else:
            n_items, arity, sp = 0, 0, None
        tb = C.create_string_buffer(tape, len(tape))
        ab = C.create_string_buffer(act_tape, len(act_tape)) if act_tape else None
        gb = C.create_string_buffer(guard_tape, len(guard_tape)) if guard_tape else None
        i = C.c_int()
        self._check(self.lib.symel_cuda_add_energy(
            self.h, name.encode(), conn, C.cast(tb, C.c_void_p), len(tape), C.cast(ins, C.c_void_p), len(inputs),
            _ptr(ds), ds.size, sp, n_items, arity,
            C.cast(ab, C.c_void_p) if ab else None, len(act_tape) if act_tape else 0, act_kind,
            C.cast(gb, C.c_void_p) if gb else None, len(guard_tape) if guard_tape else 0, C.byref(i)))
        for slot, v in (params or {}).items():
            self.set_param(i.value, slot, v)
        if flags:
            self.set_energy_flags(i.value, flags)
        self.energy_names.append(name)
        return i.value

    def set_param(self, eid: int, slot: int, value: float) -> None:
        self._check(self.lib.symel_cuda_set_param(self.h, eid, slot, float(value)))

    def set_energy_flags(self, eid: int, flags: int) -> None:
        self._check(self.lib.symel_cuda_set_energy_flags(self.h, eid, flags))

    def set_pins(self, mask: np.ndarray) -> None:
        m = np.ascontiguousarray(mask, dtype=np.uint8)
        self._check(self.lib.symel_cuda_set_pins(self.h, _ptr(m), m.size))

    # ---- assembly
    def assemble(self, mode: str = "deterministic") -> float:
        E = C.c_double()
        st = Status()
        self._check(self.lib.symel_cuda_assemble(self.h, MODES[mode], C.byref(E), C.byref(st)))
        return E.value

    def energy_only(self) -> float:
        E = C.c_double()
        self._check(self.lib.symel_cuda_energy_only(self.h, C.byref(E)))
        return E.value

    def guard_min(self) -> float:
        g = C.c_double()
        self._check(self.lib.symel_cuda_guard_min(self.h, C.byref(g)))
        return g.value

    def pattern_info(self):
        b, nr, nb, nd = C.c_int(), C.c_uint64(), C.c_uint64(), C.c_uint64()
        self._check(self.lib.symel_cuda_pattern_info(self.h, C.byref(b), C.byref(nr), C.byref(nb), C.byref(nd)))
        return b.value, nr.value, nb.value, nd.value

    def gradient(self) -> np.ndarray:
        _, _, _, nd = self.pattern_info()
        g = np.empty(nd)
        self._check(self.lib.symel_cuda_copy_gradient(self.h, _ptr(g)))
        return g

    def hessian(self) -> Bcrs:
        b, nr, nb, _ = self.pattern_info()
        rp = np.empty(nr + 1, np.int64)
        ci = np.empty(nb, np.int64)
        self._check(self.lib.symel_cuda_copy_pattern(self.h, _ptr(rp), _ptr(ci)))
        v = np.empty(nb * b * b)
        self._check(self.lib.symel_cuda_copy_hessian(self.h, _ptr(v)))
        return Bcrs(b, rp, ci, v)

    def hessian_values(self) -> np.ndarray:
        b, nr, nb, _ = self.pattern_info()
        v = np.empty(nb * b * b)
        self._check(self.lib.symel_cuda_copy_hessian(self.h, _ptr(v)))
        return v

    # ---- consumer of the assembled Hessian --------------------------------
    def matvec(self, x: np.ndarray) -> np.ndarray:
        """y = H x with the last assembled Hessian (BcrsMatrix::matvec)."""
        x = np.ascontiguousarray(x, dtype=np.float64)
        y = np.empty_like(x)
        self._check(self.lib.symel_cuda_matvec(self.h, x.ctypes.data, y.ctypes.data, 0))
        return y

    def block_jacobi(self, tau: float = 0.0) -> np.ndarray:
        """Inverses of the diagonal blocks + tau I (detail::block_jacobi_inverse), [n_rows, b, b]."""
        b, nbr, _, _ = self.pattern_info()
        inv = np.empty(nbr * b * b)
        self._check(self.lib.symel_cuda_block_jacobi(self.h, float(tau), inv.ctypes.data, 0))
        return inv.reshape(nbr, b, b)

    def pcg(self, rhs: np.ndarray, tau: float = 0.0, rel_tol: float = 1e-4, max_iters: int = 0):
        """pcg (optimizer.hpp:119-158) on (H + tau I) x = rhs; max_iters <= 0 means n_dofs (the
        Newton default, NewtonOptions::cg_max_iters). Returns (x, PcgResult as dict)."""
        rhs = np.ascontiguousarray(rhs, dtype=np.float64)
        x = np.empty_like(rhs)
        res = PcgResult()
        mi = int(max_iters) if max_iters > 0 else rhs.size
        self._check(self.lib.symel_cuda_pcg(self.h, float(tau), rhs.ctypes.data, x.ctypes.data, float(rel_tol), mi, 0,
                                            C.byref(res)))
        return x, {"iters": res.iters, "converged": bool(res.converged), "neg_curvature": bool(res.neg_curvature),
                   "rel_residual": res.rel_residual, "solve_ms": res.solve_ms}

    def gather_dofs(self) -> np.ndarray:
        """EnergySystem::gather_dofs: the flat dof vector (dof arrays in registration order)."""
        _, _, _, nd = self.pattern_info()
        u = np.empty(nd)
        self._check(self.lib.symel_cuda_gather_dofs(self.h, u.ctypes.data, 0))
        return u

    def scatter_dofs(self, u: np.ndarray) -> None:
        """EnergySystem::scatter_dofs."""
        u = np.ascontiguousarray(u, dtype=np.float64)
        self._check(self.lib.symel_cuda_scatter_dofs(self.h, u.ctypes.data, 0))

    def energy_parts(self) -> np.ndarray:
        """Per-energy energy sums of the last assemble / energy_only (energy registration order)."""
        n = len(self.energy_names)
        out = np.zeros(n)
        self._check(self.lib.symel_cuda_energy_parts(self.h, out.ctypes.data_as(C.POINTER(C.c_double)), n))
        return out

    def active_count(self, eid: int) -> int:
        n = C.c_uint64()
        self._check(self.lib.symel_cuda_active_count(self.h, eid, C.byref(n)))
        return n.value

    def element_outputs(self, eid: int, first: int, count: int, stride: int, mode: str = "deterministic"):
        out = np.empty(count * stride)
        self._check(self.lib.symel_cuda_element_outputs(self.h, eid, first, count, MODES[mode], _ptr(out)))
        return out.reshape(count, stride)

    def timings(self) -> Timings:
        t = Timings()
        self._check(self.lib.symel_cuda_get_timings(self.h, C.byref(t)))
        return t

    def launch_count(self) -> int:
        n = C.c_uint64()
        self._check(self.lib.symel_cuda_launch_count(self.h, C.byref(n)))
        return n.value

    def energy_info(self, eid: int) -> dict:
        s = EnergyStats()
        self._check(self.lib.symel_cuda_energy_info(self.h, eid, C.byref(s)))
        return {k: getattr(s, k) for k, _ in EnergyStats._fields_}

    def plan_info(self) -> dict:
        v = np.zeros(8, np.int64)
        self._check(self.lib.symel_cuda_plan_info(self.h, _ptr(v)))
        keys = ["tiles", "block_segments", "block_contributions", "block_partials", "partial_blocks",
                "row_segments", "row_partials", "partial_rows"]
        return dict(zip(keys, (int(x) for x in v)))

    def cache_stats(self) -> dict:
        """KernelCache::stats() analogue (cache.hpp:17-24) of the device kernel cache."""
        out = (C.c_uint64 * 4)()
        self._check(self.lib.symel_cuda_cache_stats(self.h, out))
        return dict(zip(("builds", "memory_hits", "disk_hits", "corrupt"), list(out)))

    def precompile(self, eid: int, mode: str = "deterministic") -> None:
        self._check(self.lib.symel_cuda_precompile(self.h, eid, MODES[mode]))

    def fp64_peak_tflops(self) -> float:
        t = C.c_double()
        self._check(self.lib.symel_cuda_fp64_peak(self.h, C.byref(t)))
        return t.value

    def stream(self) -> int:
        s = C.c_void_p()
        self._check(self.lib.symel_cuda_stream(self.h, C.byref(s)))
        return s.value or 0

    def sync(self) -> None:
        self._check(self.lib.symel_cuda_sync(self.h))

    def kernel_source(self, eid: int, mode: str = "deterministic", plan_global: bool = False) -> str:
        """Generated source; plan_global: the tile variant reading its plan slice from L2."""
        fl = MODES[mode] | (0x100 if plan_global else 0)  # SYMEL_SRC_PLAN_GLOBAL
        need = C.c_uint64()
        self._check(self.lib.symel_cuda_kernel_source(self.h, eid, fl, None, 0, C.byref(need)))
        buf = C.create_string_buffer(need.value)
        self._check(self.lib.symel_cuda_kernel_source(self.h, eid, fl, buf, need.value, None))
        return buf.value.decode()
