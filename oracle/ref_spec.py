"""TEST INFRASTRUCTURE — runs the reference's parse_synthetic_spec + generate
(oracle/_ref, io.cpp:252-399) in a process that has not loaded numpy: the
reference library carries its own static libstdc++, whose iostream locale
state must not meet another libstdc++ already loaded (parse_synthetic_spec
uses std::istringstream). Writes "<status> <count>\\n<message>\\n" + raw
doubles to the output file.

    python oracle/ref_spec.py SPEC OUT
"""
import ctypes
import os
import sys


def main(spec, out):
    here = os.path.dirname(os.path.abspath(__file__))
    L = ctypes.CDLL(os.path.join(here, "_ref", "libcheesemap_ref.so"))
    fn = L.ref_generate_spec
    fn.argtypes = [ctypes.c_char_p, ctypes.c_void_p, ctypes.c_uint64,
                   ctypes.POINTER(ctypes.c_uint64), ctypes.c_char_p, ctypes.c_int]
    fn.restype = ctypes.c_int
    n = ctypes.c_uint64()
    msg = ctypes.create_string_buffer(512)
    rc = fn(spec.encode(), None, 0, ctypes.byref(n), msg, 512)
    data = b""
    if rc == 0:
        buf = (ctypes.c_double * (3 * n.value))()
        rc = fn(spec.encode(), buf, n.value, ctypes.byref(n), msg, 512)
        data = bytes(buf)
    with open(out, "wb") as f:
        f.write(f"{rc} {n.value}\n{msg.value.decode()}\n".encode() + data)


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])
