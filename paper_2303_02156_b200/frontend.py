"""ctypes front of libsymel_host.so: tapes produced by this repo's own C++ symbolic front end
(csrc/host/symel/*.hpp), which restates the reference's differentiation pipeline and yields the
same bytes (tests/test_frontend.py checks them against the reference's own tapes)."""
import ctypes as C
import functools
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libsymel_host.so")
_lib = None


def available() -> bool:
    return os.path.exists(LIB_PATH)


def _load():
    global _lib
    if _lib is None:
        _lib = C.CDLL(LIB_PATH)
        _lib.symel_host_standard_tape.argtypes = [C.c_char_p, C.c_char_p, C.c_void_p, C.c_uint64,
                                                  C.POINTER(C.c_uint64)]
        _lib.symel_host_last_error.restype = C.c_char_p
    return _lib


@functools.lru_cache(maxsize=None)
def tape(name: str) -> bytes:
    """name: tet4_elastic | tet10_elastic | membrane | bending | inertia | contact[_act|_guard]."""
    lib = _load()
    which = "deriv"
    for suf in ("_act", "_guard"):
        if name.endswith(suf):
            name, which = name[: -len(suf)], suf[1:]
    n = C.c_uint64()
    if lib.symel_host_standard_tape(name.encode(), which.encode(), None, 0, C.byref(n)):
        raise RuntimeError(lib.symel_host_last_error().decode())
    buf = C.create_string_buffer(n.value)
    if lib.symel_host_standard_tape(name.encode(), which.encode(), buf, n.value, C.byref(n)):
        raise RuntimeError(lib.symel_host_last_error().decode())
    return buf.raw[: n.value]
