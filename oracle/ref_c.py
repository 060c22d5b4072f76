"""Call the reference's own generated CPU kernels (oracle/_ref/, built by
oracle/build_ref.py) -- TEST / BASELINE INFRASTRUCTURE ONLY.

Mirrors fevec.jit.KernelHandle.__call__(start, end, bindings)
(/root/reference/pkg/src/fevec/jit.py:71-87) without importing fevec (it
does not exist on the GPU box).  ``run_threads`` is the SURVEY.md 8d
multi-core protocol: T threads over width-aligned [start, end) chunks (the
batched targets require an aligned start, transforms.py:304-308), each with
a private dat0, summed at the end (the sum is part of the timed work);
ctypes releases the GIL during the call.
"""

import ctypes
import json
import os
from concurrent.futures import ThreadPoolExecutor

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF = os.path.join(HERE, "_ref")


def manifest():
    p = os.path.join(REF, "manifest.json")
    if not os.path.exists(p):
        return []
    with open(p) as f:
        return json.load(f)


def available(form, cell, degree, target="vector-ext"):
    return any(m["form"] == form and m["cell"] == cell and m["degree"] == degree
               and m["target"] == target for m in manifest())


class RefKernel:
    def __init__(self, form, cell, degree, target="vector-ext"):
        ms = [m for m in manifest() if m["form"] == form and m["cell"] == cell
              and m["degree"] == degree and m["target"] == target]
        if not ms:
            raise FileNotFoundError(f"no reference kernel for {form} {cell} p{degree} {target}")
        self.m = ms[0]
        self.width = self.m["width"]
        lib = ctypes.CDLL(os.path.join(REF, self.m["so"]))
        self.fn = getattr(lib, self.m["entry"])
        argt = []
        for a in self.m["args"]:
            if a in ("start", "end"):
                argt.append(ctypes.c_int32)
            elif a.startswith("map"):
                argt.append(ctypes.POINTER(ctypes.c_int32))
            else:
                argt.append(ctypes.POINTER(ctypes.c_double))
        self.fn.argtypes = argt
        self.fn.restype = None
        self._lib = lib

    def __call__(self, start, end, bindings):
        args = [ctypes.c_int32(start), ctypes.c_int32(end)]
        for a in self.m["args"][2:]:
            buf = bindings[a]
            t = ctypes.c_int32 if a.startswith("map") else ctypes.c_double
            args.append(buf.ctypes.data_as(ctypes.POINTER(t)))
        self.fn(*args)

    def run_threads(self, ncells, bindings, threads, start=0):
        """Cells [start, ncells) on `threads` threads with private outputs
        (chunk starts width-aligned relative to start, which must itself be
        width-aligned); returns y."""
        w = self.width
        if start % w:
            raise ValueError(f"start {start} is not a multiple of the SIMD width {w}")
        n = ncells - start
        chunk = -(-n // threads)
        chunk = -(-chunk // w) * w
        cuts = list(range(start, ncells, chunk)) + [ncells]
        outs = [np.zeros_like(bindings["dat0"]) for _ in cuts[:-1]]

        def work(i):
            b = dict(bindings)
            b["dat0"] = outs[i]
            self(cuts[i], cuts[i + 1], b)

        with ThreadPoolExecutor(len(outs)) as ex:
            list(ex.map(work, range(len(outs))))
        y = outs[0]
        for o in outs[1:]:
            y += o
        return y
