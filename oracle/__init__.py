"""TEST INFRASTRUCTURE ONLY — ctypes access to the CPU checkers.

* ``orc()``  — our C restatement (oracle/liborc.so, oracle/ccd_oracle.c).
* ``ref()``  — the UNMODIFIED reference compiled from /root/reference by
  oracle/Makefile into oracle/_ref/libccdref.so (with oracle/ref_adapter.cpp).

Only tests/, __graft_entry__.smoke() and bench.py's reference/cpu_baseline leg
may import this package.  The product never does.  Both libraries are built
in the dev container and shipped prebuilt to the GPU box (which has no
/root/reference).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

from paper_2112_06300_b200 import abi
from paper_2112_06300_b200.abi import P_F32, P_F64, P_U8, P_U16, P_U32, P_U64, ptr

HERE = os.path.dirname(os.path.abspath(__file__))
ORC_SO = os.path.join(HERE, "liborc.so")
REF_SO = os.path.join(HERE, "_ref", "libccdref.so")
REFERENCE_SRC = "/root/reference/proj/src"


def build(force: bool = False) -> None:
    """Build liborc.so always, libccdref.so when the reference sources exist."""
    targets = ["liborc.so"]
    if os.path.isdir(REFERENCE_SRC):
        targets.append("ref")
    if force:
        subprocess.run(["make", "-C", HERE, "clean"], check=True, capture_output=True)
    subprocess.run(["make", "-C", HERE, "-j8"] + targets, check=True, capture_output=True)


class CheckerError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"[{code}] {msg}")
        self.code = code


class _Cpu:
    """Common numpy-level interface over liborc / libccdref."""

    def __init__(self, path: str, prefix: str, threads: int = 1):
        if not os.path.exists(path):
            raise FileNotFoundError(path)
        self.lib = C.CDLL(path)
        self.prefix = prefix
        self.threads = threads
        self.is_ref = prefix == "ref"

    def fn(self, name):
        return getattr(self.lib, f"{self.prefix}_{name}")

    def _check(self, rc):
        if rc != 0:
            msg = ""
            if self.is_ref:
                self.lib.ref_last_error.restype = C.c_char_p
                msg = self.lib.ref_last_error().decode()
            raise CheckerError(rc, msg)

    def _take(self, p, n, dtype):
        if n == 0:
            out = np.zeros(0, dtype)
        else:
            out = np.ctypeslib.as_array(C.cast(p, C.POINTER(np.ctypeslib.as_ctypes_type(dtype))),
                                        shape=(n,)).copy()
        (self.lib.ref_free if self.is_ref else self.lib.orc_free)(p)
        return out

    # ---- geometry
    def round_reduced(self, x: np.ndarray):
        x = np.ascontiguousarray(x, np.float64)
        d = np.empty(x.size, np.float32)
        u = np.empty(x.size, np.float32)
        if self.is_ref:
            self._check(self.lib.ref_round(ptr(x, C.c_double), C.c_uint64(x.size),
                                           ptr(d, C.c_float), ptr(u, C.c_float)))
        else:
            self.lib.orc_round_down_reduced.restype = C.c_float
            self.lib.orc_round_up_reduced.restype = C.c_float
            for i, v in enumerate(x):
                d[i] = self.lib.orc_round_down_reduced(C.c_double(v))
                u[i] = self.lib.orc_round_up_reduced(C.c_double(v))
        return d, u

    def build_boxes(self, s, inflation=0.0):
        k = s.primitive_count()
        mn = np.empty((k, 3), np.float32)
        mx = np.empty((k, 3), np.float32)
        kind = np.empty(k, np.uint8)
        idx = np.empty(k, np.uint32)
        args = [ptr(s.vertices_t0, C.c_double), ptr(s.vertices_t1, C.c_double), C.c_uint64(s.nv),
                ptr(s.edges, C.c_uint32), C.c_uint64(s.ne), ptr(s.faces, C.c_uint32),
                C.c_uint64(s.nf), C.c_double(inflation)]
        if self.is_ref:
            args.append(C.c_uint(self.threads))
        args += [ptr(mn, C.c_float), ptr(mx, C.c_float), ptr(kind, C.c_uint8), ptr(idx, C.c_uint32)]
        self._check(self.fn("build_boxes")(*args))
        return mn, mx, kind, idx

    def choose_axis(self, mn, mx):
        mn = np.ascontiguousarray(mn, np.float32)
        mx = np.ascontiguousarray(mx, np.float32)
        if self.is_ref:
            a = C.c_int()
            self._check(self.lib.ref_choose_axis(ptr(mn, C.c_float), ptr(mx, C.c_float),
                                                 C.c_uint64(mn.shape[0]), C.byref(a)))
            return a.value
        return self.lib.orc_choose_axis(ptr(mn, C.c_float), ptr(mx, C.c_float),
                                        C.c_uint64(mn.shape[0]))

    def broad(self, method, boxes, s, rb=0, re=abi.UINT64_MAX):
        """Returns (pairs (n,2) u64, round_sizes u64[], max_queue)."""
        mn, mx, kind, idx = [np.ascontiguousarray(a) for a in boxes]
        k = mn.shape[0]
        pp, npairs = P_U64(), C.c_uint64()
        rp, nr, mq = P_U64(), C.c_uint64(), C.c_uint64()
        if self.is_ref:
            self._check(self.lib.ref_broad(
                C.c_int(method), ptr(mn, C.c_float), ptr(mx, C.c_float), ptr(kind, C.c_uint8),
                ptr(idx, C.c_uint32), C.c_uint64(k), ptr(s.vertices_t0, C.c_double),
                ptr(s.vertices_t1, C.c_double), C.c_uint64(s.nv), ptr(s.edges, C.c_uint32),
                C.c_uint64(s.ne), ptr(s.faces, C.c_uint32), C.c_uint64(s.nf),
                C.c_uint(self.threads), C.c_uint64(rb), C.c_uint64(re), C.byref(pp),
                C.byref(npairs), C.byref(rp), C.byref(nr), C.byref(mq)))
        else:
            self._check(self.lib.orc_broad(
                C.c_int(method), ptr(mn, C.c_float), ptr(mx, C.c_float), ptr(kind, C.c_uint8),
                ptr(idx, C.c_uint32), C.c_uint64(k), ptr(s.edges, C.c_uint32), C.c_uint64(s.ne),
                ptr(s.faces, C.c_uint32), C.c_uint64(s.nf), C.c_uint64(rb), C.c_uint64(re),
                C.byref(pp), C.byref(npairs), C.byref(rp), C.byref(nr), C.byref(mq)))
        pairs = self._take(pp, 2 * npairs.value, np.uint64).reshape(-1, 2)
        rounds = self._take(rp, nr.value, np.uint64) if rp else np.zeros(0, np.uint64)
        return pairs, rounds, mq.value

    def classify(self, pairs, s):
        pairs = np.ascontiguousarray(pairs, np.uint64).reshape(-1, 2)
        n = pairs.shape[0]
        kind = np.empty(max(n, 1), np.uint8)
        pts = np.empty((max(n, 1), 24), np.float64)
        src = np.empty((max(n, 1), 2), np.uint64)
        nvf, nee = C.c_uint64(), C.c_uint64()
        self._check(self.fn("classify")(
            ptr(pairs, C.c_uint64), C.c_uint64(n), ptr(s.vertices_t0, C.c_double),
            ptr(s.vertices_t1, C.c_double), C.c_uint64(s.nv), ptr(s.edges, C.c_uint32),
            C.c_uint64(s.ne), ptr(s.faces, C.c_uint32), C.c_uint64(s.nf), ptr(kind, C.c_uint8),
            ptr(pts, C.c_double), ptr(src, C.c_uint64), C.byref(nvf), C.byref(nee)))
        m = nvf.value + nee.value
        return kind[:m].copy(), pts[:m].copy(), src[:m].copy(), nvf.value

    # ---- narrow phase
    def inclusion_box(self, kind, points, box):
        points = np.ascontiguousarray(points, np.float64)
        box = np.ascontiguousarray(box, np.float64)
        out = np.empty(6, np.float64)
        if self.is_ref:
            self._check(self.lib.ref_inclusion_box(C.c_uint8(kind), ptr(points, C.c_double),
                                                   ptr(box, C.c_double), ptr(out, C.c_double)))
        else:
            self.lib.orc_inclusion_box(C.c_uint8(kind), ptr(points, C.c_double),
                                       ptr(box, C.c_double), ptr(out, C.c_double))
        return out

    def process_interval(self, kind, points, box, depth, t_star, sep, cfg):
        points = np.ascontiguousarray(points, np.float64)
        box = np.ascontiguousarray(box, np.float64)
        depth = np.ascontiguousarray(depth, np.uint16)
        action, zd = C.c_uint8(), C.c_uint8()
        ct = C.c_double()
        ch = np.zeros(12, np.float64)
        cd = np.zeros(6, np.uint16)
        args = [C.c_uint8(kind), ptr(points, C.c_double), ptr(box, C.c_double),
                ptr(depth, C.c_uint16), C.c_double(t_star), C.c_double(sep), C.byref(cfg),
                C.byref(action), C.byref(ct), C.byref(zd), ptr(ch, C.c_double),
                ptr(cd, C.c_uint16)]
        if self.is_ref:
            self._check(self.lib.ref_process_interval(*args))
        else:
            self.lib.orc_process_interval(*args)
        return action.value, ct.value, zd.value, ch, cd

    def narrow_phase(self, kind, points, cfg, capacity=abi.UINT64_MAX, seps=None):
        kind = np.ascontiguousarray(kind, np.uint8)
        points = np.ascontiguousarray(points, np.float64)
        n = kind.size
        toi = np.empty(max(n, 1), np.float64)
        flags = np.empty(max(n, 1), np.uint8)
        st = abi.NarrowStats()
        seps_p = ptr(np.ascontiguousarray(seps, np.float64), C.c_double) if seps is not None else None
        if self.is_ref:
            self._check(self.lib.ref_narrow_phase(
                ptr(kind, C.c_uint8), ptr(points, C.c_double), C.c_uint64(n), seps_p, C.byref(cfg),
                C.c_uint(self.threads), C.c_uint64(capacity), ptr(toi, C.c_double),
                ptr(flags, C.c_uint8), C.byref(st)))
        else:
            self._check(self.lib.orc_narrow_phase(
                ptr(kind, C.c_uint8), ptr(points, C.c_double), C.c_uint64(n), seps_p, C.byref(cfg),
                C.c_uint64(capacity), ptr(toi, C.c_double), ptr(flags, C.c_uint8), C.byref(st)))
        return toi[:n].copy(), flags[:n].copy(), st

    def ccd(self, s, cfg, no_zero_retry=False, want_pairs=True):
        rep = abi.Report()
        pp = P_U64()
        args = [ptr(s.vertices_t0, C.c_double), ptr(s.vertices_t1, C.c_double), C.c_uint64(s.nv),
                ptr(s.edges, C.c_uint32), C.c_uint64(s.ne), ptr(s.faces, C.c_uint32),
                C.c_uint64(s.nf), C.byref(cfg)]
        if self.is_ref:
            args.append(C.c_int(int(no_zero_retry)))
        args += [C.byref(rep), C.byref(pp) if want_pairs else None]
        self._check(self.fn("ccd")(*args))
        pairs = self._take(pp, 2 * rep.candidate_count, np.uint64).reshape(-1, 2) if want_pairs else None
        return rep, pairs

    # ---- reference-only helpers
    def run_batched(self, s, boxes, cfg):
        """run_batched (pipeline.cpp:179-215) on a caller's box list.
        Returns (report, pairs (n,2) u64, broad_batches, narrow_batches)."""
        mn, mx, kind, idx = [np.ascontiguousarray(a) for a in boxes]
        rep = abi.Report()
        pp, bb, nb = P_U64(), C.c_uint64(), C.c_uint64()
        self._check(self.lib.ref_run_batched(
            ptr(s.vertices_t0, C.c_double), ptr(s.vertices_t1, C.c_double), C.c_uint64(s.nv),
            ptr(s.edges, C.c_uint32), C.c_uint64(s.ne), ptr(s.faces, C.c_uint32), C.c_uint64(s.nf),
            ptr(mn, C.c_float), ptr(mx, C.c_float), ptr(kind, C.c_uint8), ptr(idx, C.c_uint32),
            C.c_uint64(mn.shape[0]), C.byref(cfg), C.byref(rep), C.byref(bb), C.byref(nb), C.byref(pp)))
        pairs = self._take(pp, 2 * rep.candidate_count, np.uint64).reshape(-1, 2)
        return rep, pairs, bb.value, nb.value

    def make_scene(self, name, *args):
        from paper_2112_06300_b200.scenes import SceneStep
        v0, v1, e, f = P_F64(), P_F64(), P_U32(), P_U32()
        nv, ne, nf = C.c_uint64(), C.c_uint64(), C.c_uint64()
        fn = {"cloth": self.lib.ref_make_cloth_scene, "soup": self.lib.ref_make_box_soup}[name]
        if name == "cloth":
            a = [C.c_uint64(args[0]), C.c_uint64(args[1]), C.c_double(args[2]), C.c_double(args[3]),
                 C.c_uint64(args[4])]
        else:
            a = [C.c_uint64(args[0]), C.c_double(args[1]), C.c_double(args[2]), C.c_double(args[3]),
                 C.c_uint64(args[4])]
        self._check(fn(*a, C.byref(v0), C.byref(v1), C.byref(nv), C.byref(e), C.byref(ne),
                       C.byref(f), C.byref(nf)))
        return SceneStep(self._take(v0, 3 * nv.value, np.float64),
                         self._take(v1, 3 * nv.value, np.float64),
                         self._take(e, 2 * ne.value, np.uint32),
                         self._take(f, 3 * nf.value, np.uint32))

    def query_min_separations(self, kind, points, pcfg):
        kind = np.ascontiguousarray(kind, np.uint8)
        points = np.ascontiguousarray(points, np.float64)
        out = np.empty(max(kind.size, 1))
        self._check(self.lib.ref_query_min_separations(ptr(kind, C.c_uint8), ptr(points, C.c_double),
                                                       C.c_uint64(kind.size), C.byref(pcfg),
                                                       ptr(out, C.c_double)))
        return out[:kind.size].copy()


_cache = {}


def orc() -> _Cpu:
    if "orc" not in _cache:
        if not os.path.exists(ORC_SO):
            build()
        _cache["orc"] = _Cpu(ORC_SO, "orc")
    return _cache["orc"]


def ref_available() -> bool:
    return os.path.exists(REF_SO)


def ref(threads: int = 1) -> _Cpu:
    key = ("ref", threads)
    if key not in _cache:
        if not os.path.exists(REF_SO) and os.path.isdir(REFERENCE_SRC):
            build()
        _cache[key] = _Cpu(REF_SO, "ref", threads)
    return _cache[key]
