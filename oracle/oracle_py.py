"""Python access to the oracles -- TEST INFRASTRUCTURE ONLY.

Two checkers live here:
  * ``COracle``: ctypes binding of oracle/libwmc_oracle.so, our plain-C
    restatement of the reference hot path (oracle/wmc_oracle.c);
  * ``RefDriver``: the unmodified reference library composed by
    oracle/ref_driver.cpp into oracle/_ref/wavemc_ref_driver.
Only tests/, __graft_entry__.smoke() and bench.py (cpu_baseline / --impl
reference) use this module; the product package never imports it.
"""
from __future__ import annotations

import ctypes as C
import json
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "libwmc_oracle.so")
REF_DRIVER = os.path.join(HERE, "_ref", "wavemc_ref_driver")


class OMesh(C.Structure):
    _fields_ = [("n_vertices", C.c_int), ("n_triangles", C.c_int), ("xy", C.POINTER(C.c_double)),
                ("tri", C.POINTER(C.c_int)), ("fine", C.POINTER(C.c_ubyte)), ("boundary", C.POINTER(C.c_ubyte))]


class OProblem(C.Structure):
    _fields_ = [("cells_x", C.c_int), ("cells_y", C.c_int), ("coef_lo", C.c_double), ("coef_hi", C.c_double),
                ("final_time", C.c_double), ("dt", C.c_double), ("substeps", C.c_int), ("nu", C.c_double),
                ("kind", C.c_int), ("ic_x", C.c_double), ("ic_y", C.c_double), ("ic_w2", C.c_double),
                ("box", C.c_double * 4), ("kl_table", C.POINTER(C.c_double)), ("kl_modes", C.c_int),
                ("tiers", C.c_int), ("domain", C.c_double * 4), ("qoi_mean", C.c_int),
                ("cfl_safety", C.c_double), ("warm_full", C.POINTER(C.c_double)),
                ("warm_coarse", C.POINTER(C.c_double))]


def build(force: bool = False) -> None:
    """Compile the C restatement (and, when /root/reference exists, the
    reference driver) with oracle/Makefile."""
    targets = ["oracle"]
    if os.path.isdir("/root/reference/proj/src"):
        targets.append("ref")
    if force or not os.path.exists(ORACLE_SO) or ("ref" in targets and not os.path.exists(REF_DRIVER)):
        subprocess.run(["make", "-C", HERE] + targets, check=True, capture_output=True)


class MeshArrays:
    """Keeps numpy arrays alive behind an OMesh."""

    def __init__(self, xy, tri, fine, boundary):
        self.xy = np.ascontiguousarray(xy, np.float64)
        self.tri = np.ascontiguousarray(tri, np.int32)
        self.fine = np.ascontiguousarray(fine, np.uint8)
        self.boundary = np.ascontiguousarray(boundary, np.uint8)
        self.c = OMesh(len(self.xy), len(self.tri), self.xy.ctypes.data_as(C.POINTER(C.c_double)),
                       self.tri.ctypes.data_as(C.POINTER(C.c_int)), self.fine.ctypes.data_as(C.POINTER(C.c_ubyte)),
                       self.boundary.ctypes.data_as(C.POINTER(C.c_ubyte)))


def problem(dt, substeps=1, kind=1, final_time=1.0, nu=0.01, cells=(4, 4), coef=(0.5, 1.5),
            ic=(0.3, 0.5, 0.01), box=(0.7, 0.9, 0.4, 0.6), kl_table=None, tiers=1, domain=None,
            qoi_mean=False, cfl_safety=0.0) -> OProblem:
    """kl_table: None (uniform cells) or a contiguous float64 array [cell][mode]
    (kept alive by the returned struct)."""
    p = OProblem()
    if kl_table is not None:
        kl_table = np.ascontiguousarray(kl_table, np.float64)
        p._kl_keep = kl_table
        p.kl_table = kl_table.ctypes.data_as(C.POINTER(C.c_double))
        p.kl_modes = kl_table.shape[1]
    p.cells_x, p.cells_y = cells
    p.coef_lo, p.coef_hi = coef
    p.final_time, p.dt, p.substeps, p.nu, p.kind = final_time, dt, substeps, nu, kind
    p.ic_x, p.ic_y, p.ic_w2 = ic
    for i, v in enumerate(box):
        p.box[i] = v
    p.tiers = tiers
    if domain is not None:
        for i, v in enumerate(domain):
            p.domain[i] = v
    p.qoi_mean = 1 if qoi_mean else 0
    p.cfl_safety = cfl_safety
    return p


class COracle:
    def __init__(self):
        if not os.path.exists(ORACLE_SO):
            build()
        self.lib = C.CDLL(ORACLE_SO)
        L = self.lib
        L.wmc_oracle_mix64.restype = C.c_uint64
        L.wmc_oracle_mix64.argtypes = [C.c_uint64]
        L.wmc_oracle_stream_words.argtypes = [C.c_uint64, C.c_uint32, C.c_uint64, C.c_int, C.POINTER(C.c_uint64)]
        L.wmc_oracle_draw_cells.argtypes = [C.c_uint64, C.c_uint32, C.c_uint64, C.c_int, C.c_double, C.c_double,
                                            C.POINTER(C.c_double)]
        L.wmc_oracle_draw_kl.argtypes = [C.c_uint64, C.c_uint32, C.c_uint64, C.POINTER(C.c_double), C.c_int,
                                         C.c_int, C.POINTER(C.c_double)]
        L.wmc_oracle_chebyshev.argtypes = [C.c_int, C.c_double, C.POINTER(C.c_double), C.POINTER(C.c_double),
                                           C.POINTER(C.c_double), C.POINTER(C.c_double)]
        L.wmc_oracle_solve.argtypes = [C.POINTER(OMesh), C.POINTER(OProblem), C.POINTER(C.c_double),
                                       C.POINTER(C.c_double), C.POINTER(C.c_long), C.POINTER(C.c_long)]
        L.wmc_oracle_eval_pairs.argtypes = [C.POINTER(OMesh), C.POINTER(OProblem), C.POINTER(OMesh),
                                            C.POINTER(OProblem), C.c_uint64, C.c_uint32, C.c_uint64, C.c_long,
                                            C.POINTER(C.c_double), C.POINTER(C.c_double), C.POINTER(C.c_long),
                                            C.POINTER(C.c_long)]
        L.wmc_oracle_steps.argtypes = [C.POINTER(OMesh), C.POINTER(OProblem), C.POINTER(C.c_double),
                                       C.POINTER(C.c_double), C.POINTER(C.c_double), C.c_long]
        L.wmc_oracle_stable_dt.argtypes = [C.POINTER(OMesh), C.POINTER(OProblem), C.POINTER(C.c_double),
                                           C.POINTER(C.c_double), C.POINTER(C.c_int)]
        L.wmc_oracle_warm_starts.argtypes = [C.POINTER(OMesh), C.POINTER(OProblem), C.POINTER(C.c_double),
                                             C.POINTER(C.c_double)]
        L.wmc_oracle_moments.argtypes = [C.POINTER(C.c_double), C.POINTER(C.c_double), C.c_long,
                                         C.POINTER(C.c_double)]
        L.wmc_oracle_level_data.argtypes = [C.POINTER(OMesh), C.POINTER(OProblem), C.POINTER(C.c_double),
                                            C.POINTER(C.c_double), C.POINTER(C.c_double)]

    def stream_words(self, seed, level, index, count):
        out = (C.c_uint64 * count)()
        self.lib.wmc_oracle_stream_words(seed, level, index, count, out)
        return [int(v) for v in out]

    def draw_cells(self, seed, level, index, n_cells=16, lo=0.5, hi=1.5):
        out = np.empty(n_cells, np.float64)
        self.lib.wmc_oracle_draw_cells(seed, level, index, n_cells, lo, hi, out.ctypes.data_as(C.POINTER(C.c_double)))
        return out

    def draw_kl(self, seed, level, index, table):
        table = np.ascontiguousarray(table, np.float64)
        out = np.empty(table.shape[0], np.float64)
        self.lib.wmc_oracle_draw_kl(seed, level, index, table.ctypes.data_as(C.POINTER(C.c_double)), table.shape[0],
                                    table.shape[1], out.ctypes.data_as(C.POINTER(C.c_double)))
        return out

    def chebyshev(self, p, nu):
        d, o = C.c_double(), C.c_double()
        bi = (C.c_double * max(p, 1))()
        bh = (C.c_double * max(p, 1))()
        rc = self.lib.wmc_oracle_chebyshev(p, nu, C.byref(d), C.byref(o), bi, bh)
        if rc:
            raise ValueError("chebyshev_constants: bad arguments")
        return d.value, o.value, list(bi)[: p - 1], list(bh)[: p - 1]

    def solve(self, mesh: MeshArrays, pb: OProblem, cells):
        cells = np.ascontiguousarray(cells, np.float64)
        q = C.c_double()
        step = C.c_long()
        cnt = (C.c_long * 3)()
        rc = self.lib.wmc_oracle_solve(C.byref(mesh.c), C.byref(pb), cells.ctypes.data_as(C.POINTER(C.c_double)),
                                       C.byref(q), C.byref(step), cnt)
        return rc, q.value, step.value, list(cnt)

    def stable_dt(self, mesh: MeshArrays, pb: OProblem, cells):
        """Reference stable_dt of one sample: (status, dt, [full iters, coarse iters])."""
        cells = np.ascontiguousarray(cells, np.float64)
        dt = C.c_double()
        it = (C.c_int * 2)()
        rc = self.lib.wmc_oracle_stable_dt(C.byref(mesh.c), C.byref(pb), cells.ctypes.data_as(C.POINTER(C.c_double)),
                                           C.byref(dt), it)
        return rc, dt.value, list(it)

    def warm_starts(self, mesh: MeshArrays, pb: OProblem):
        n = int((mesh.boundary == 0).sum())
        wf, wc = np.empty(n), np.empty(n)
        rc = self.lib.wmc_oracle_warm_starts(C.byref(mesh.c), C.byref(pb), wf.ctypes.data_as(C.POINTER(C.c_double)),
                                             wc.ctypes.data_as(C.POINTER(C.c_double)))
        return rc, wf, wc

    def steps(self, mesh: MeshArrays, pb: OProblem, cells, z_prev, z_curr, n_steps):
        """Advance a consistent pair (z_prev, z_curr) by n_steps (no start-up step)."""
        cells = np.ascontiguousarray(cells, np.float64)
        zp = np.array(z_prev, np.float64)
        zc = np.array(z_curr, np.float64)
        rc = self.lib.wmc_oracle_steps(C.byref(mesh.c), C.byref(pb), cells.ctypes.data_as(C.POINTER(C.c_double)),
                                       zp.ctypes.data_as(C.POINTER(C.c_double)),
                                       zc.ctypes.data_as(C.POINTER(C.c_double)), n_steps)
        return rc, zp, zc

    def eval_pairs(self, fine: MeshArrays, pf: OProblem, coarse: MeshArrays | None, pc: OProblem | None, seed,
                   level, first, count):
        dq = np.empty(count, np.float64)
        qf = np.empty(count, np.float64)
        fi, fs = C.c_long(-1), C.c_long(0)
        rc = self.lib.wmc_oracle_eval_pairs(C.byref(fine.c), C.byref(pf), C.byref(coarse.c) if coarse else None,
                                            C.byref(pc) if pc else None, seed, level, first, count,
                                            dq.ctypes.data_as(C.POINTER(C.c_double)),
                                            qf.ctypes.data_as(C.POINTER(C.c_double)), C.byref(fi), C.byref(fs))
        return rc, dq, qf, fi.value, fs.value

    def moments(self, dq, q):
        dq = np.ascontiguousarray(dq, np.float64)
        q = np.ascontiguousarray(q, np.float64)
        out = np.empty(7, np.float64)
        self.lib.wmc_oracle_moments(dq.ctypes.data_as(C.POINTER(C.c_double)), q.ctypes.data_as(C.POINTER(C.c_double)),
                                    len(dq), out.ctypes.data_as(C.POINTER(C.c_double)))
        return dict(zip(["n", "sum_dq", "sum_dq2", "sum_q", "sum_q2", "variance", "mc_variance"], out.tolist()))

    def level_data(self, mesh: MeshArrays, pb: OProblem):
        n = int((mesh.boundary == 0).sum())
        z0, mass, w = (np.empty(n, np.float64) for _ in range(3))
        got = self.lib.wmc_oracle_level_data(C.byref(mesh.c), C.byref(pb), z0.ctypes.data_as(C.POINTER(C.c_double)),
                                             mass.ctypes.data_as(C.POINTER(C.c_double)),
                                             w.ctypes.data_as(C.POINTER(C.c_double)))
        assert got == n
        return z0, mass, w


class RefDriver:
    """The reference library through oracle/_ref/wavemc_ref_driver."""

    def __init__(self, path: str = REF_DRIVER):
        if not os.path.exists(path):
            raise FileNotFoundError(f"reference driver not built: {path} (oracle/Makefile ref)")
        self.path = path

    def run(self, *args, timeout=3600) -> str:
        r = subprocess.run([self.path, *map(str, args)], capture_output=True, text=True, timeout=timeout)
        if r.returncode != 0:
            raise RuntimeError(f"ref driver {args[0]} failed ({r.returncode}): {r.stderr.strip()}")
        return r.stdout

    def solve(self, mesh_path, dt, p, kind="lts", stream_level=0, first=0, count=1, threads=0, **kw):
        out = self.run("solve", "--level-spec", f"{mesh_path},{dt!r},{p}", "--kind", kind, "--stream-level",
                       stream_level, "--first", first, "--count", count, "--threads", threads,
                       *sum(([f"--{k}", v] for k, v in kw.items()), []))
        lines = out.strip().splitlines()
        header = dict(kv.split("=") for kv in lines[0][2:].split())
        q = np.array([float(l.split()[1]) for l in lines[1:]])
        return header, q

    def mlmc(self, specs, counts, kind="lts", threads=0, per_sample=False, seed=0, timeout=3600, **kw):
        args = ["mlmc", "--kind", kind, "--N", ",".join(map(str, counts)), "--threads", threads, "--seed", seed]
        for mesh_path, dt, p in specs:
            args += ["--level-spec", f"{mesh_path},{dt!r},{p}"]
        if per_sample:
            args += ["--per-sample", 1]
        for k, v in kw.items():
            args += [f"--{k}", v]
        return json.loads(self.run(*args, timeout=timeout))

    def adaptive(self, specs, eps, threads=0, seed=0, max_level=6, kind="lts", **kw):
        """Reference run_mlmc (src/mlmc.cpp:165-233) over the given levels."""
        args = ["adaptive", "--kind", kind, "--eps", repr(eps), "--threads", threads, "--seed", seed,
                "--max-level", max_level]
        for mesh_path, dt, p in specs:
            args += ["--level-spec", f"{mesh_path},{dt!r},{p}"]
        for k, v in kw.items():
            args += [f"--{k}", v]
        return json.loads(self.run(*args))

    def level(self, mesh_path, dt, p, kind="lts"):
        out = self.run("level", "--level-spec", f"{mesh_path},{dt!r},{p}", "--kind", kind)
        rows = [l.split() for l in out.strip().splitlines()[1:]]
        return (np.array([int(r[0]) for r in rows]), np.array([float(r[1]) for r in rows]),
                np.array([float(r[2]) for r in rows]), np.array([float(r[3]) for r in rows]))

    def rng(self, seed, level, index, count, uniform=False):
        out = self.run("rng", "--seed", seed, "--level", level, "--index", index, "--count", count,
                       "--uniform", int(uniform))
        return [float(v) if uniform else int(v, 16) for v in out.split()]

    def consts(self, p, nu):
        rows = [list(map(float, l.split())) for l in self.run("consts", "--p", p, "--nu", repr(nu)).strip().splitlines()]
        return rows[0][0], rows[0][1], [r[0] for r in rows[1:]], [r[1] for r in rows[1:]]

    def experiment(self, name, kind="lts", level=None, first=0, count=1, eps=None, threads=0, **kw):
        """The reference's own sampling experiment via make_problem (src/experiments.cpp:194-237)."""
        args = ["experiment", "--name", name, "--kind", kind, "--threads", threads]
        if level is not None:
            args += ["--level", level, "--first", first, "--count", count]
        if eps is not None:
            args += ["--eps", repr(eps)]
        for k, v in kw.items():
            args += [f"--{k}", v]
        return json.loads(self.run(*args))

    def meshcheck(self, mesh_path):
        return json.loads(self.run("meshcheck", "--mesh", mesh_path))
