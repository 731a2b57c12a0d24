"""Convergence harness and command-line front end (`cli_harness`).

The reference's console script `stfem = "stfem.cli:main"` (pkg/pyproject.toml:15-16)
names this module but the snapshot does not ship it.  This is
the §8(f) rank-4 row: a thin orchestration layer over the GPU path that
reproduces the structure of the paper's Tables 1-3.

  run_convergence(RunConfig) -> [ConvergenceRow]
  emit(rows, "table" | "csv") -> str
  parse_csv(text) -> [ConvergenceRow]               (round-trip oracle)
  RunConfig.parse(text) / .serialize()              flat key=value
  main(argv)                                        subcommands solve | convergence;
                                                    exit 0 ok, 2 solver failure, 3 config error

Per level J the spatial mesh is refined J times (square:<m> -> square(m 2^J),
the same triangulation refine_uniform produces), the temporal mesh has
N_t = nt 2^J elements (uniform or graded), the operators and the load vector
are assembled on the GPU (K1/K2), the FD or BS solve runs on the GPU, and the
space-time errors are integrated on the GPU (K8).  Timing excludes assembly
 and includes steps 1-4.
"""

from __future__ import annotations

import argparse
import math
import sys
from dataclasses import asdict, dataclass, fields

import numpy as np

HEADER = "n,hx,ht,errL2,eocL2,errH1,eocH1,solve_s,kappa2"
PROBLEMS = ("paper", "sinpit", "texp", "zero")


class ConfigError(ValueError):
    """Invalid run configuration (exit code 3)."""


@dataclass
class RunConfig:
    """SPEC.md:491-494.  spatial: square:<m> | lshape:<n>; temporal: uniform |
    graded:<q>; problem: a manufactured solution (paper / sinpit / texp) or
    zero (f = 0, psi0 = 0); mem_guard_gib: refuse levels whose estimated peak
    (n complex values x 6 device arrays) exceeds it."""

    spatial: str = "square:32"
    temporal: str = "uniform"
    T: float = 5.0
    nt: int = 64
    levels: int = 0
    solver: str = "fd"
    threads: int = 1
    problem: str = "paper"
    out: str = ""
    format: str = "table"
    mem_guard_gib: float = 8.0

    def validate(self) -> "RunConfig":
        kind, _, arg = self.spatial.partition(":")
        if kind not in ("square", "lshape") or not arg.isdigit() or int(arg) < 2:
            raise ConfigError(f"spatial preset {self.spatial!r}: expected square:<m> or lshape:<n>, m >= 2")
        if self.temporal != "uniform":
            k, _, q = self.temporal.partition(":")
            try:
                qv = float(q)
            except ValueError:
                qv = float("nan")
            if k != "graded" or not qv >= 1.0:
                raise ConfigError(f"temporal preset {self.temporal!r}: expected uniform or graded:<q>, q >= 1")
        if not (self.T > 0 and self.nt >= 1 and self.levels >= 0 and self.threads >= 1):
            raise ConfigError("T > 0, nt >= 1, levels >= 0 and threads >= 1 required")
        if self.solver not in ("fd", "bs"):
            raise ConfigError(f"solver {self.solver!r}: expected fd or bs")
        if self.problem not in PROBLEMS:
            raise ConfigError(f"problem {self.problem!r}: expected one of {PROBLEMS}")
        if self.format not in ("table", "csv"):
            raise ConfigError(f"format {self.format!r}: expected table or csv")
        if not self.mem_guard_gib > 0:
            raise ConfigError("mem_guard_gib must be positive")
        return self

    def serialize(self) -> str:
        return "".join(f"{f.name}={getattr(self, f.name)}\n" for f in fields(self))

    @classmethod
    def parse(cls, text: str) -> "RunConfig":
        """Flat key=value lines; '#' starts a comment."""
        kw = {}
        types = {f.name: f.type for f in fields(cls)}
        for ln, line in enumerate(text.splitlines(), 1):
            line = line.split("#", 1)[0].strip()
            if not line:
                continue
            key, sep, val = line.partition("=")
            key, val = key.strip(), val.strip()
            if not sep or key not in types:
                raise ConfigError(f"config line {ln}: unknown or malformed entry {line!r}")
            try:
                kw[key] = {"float": float, "int": int}.get(types[key], str)(val)
            except ValueError as exc:
                raise ConfigError(f"config line {ln}: {exc}") from exc
        return cls(**kw).validate()


@dataclass
class ConvergenceRow:
    """SPEC.md:496-499 (Table 1/2/3 column layout)."""

    n: int
    hx: float
    ht: float
    errL2: float
    eocL2: float | None
    errH1: float
    eocH1: float | None
    solve_s: float
    kappa2: float


def _fmt(v) -> str:
    return "-" if v is None else f"{v:.3e}"   # 4 significant digits


def emit(rows, fmt: str = "table") -> str:
    """CSV with HEADER, scientific notation with 4 significant
    digits, '-' for the first row's eoc; the table mirrors the paper's columns."""
    if not rows:
        raise ValueError("emit: no rows")
    if fmt == "csv":
        out = [HEADER]
        for r in rows:
            out.append(",".join([str(r.n)] + [_fmt(getattr(r, k)) for k in HEADER.split(",")[1:]]))
        return "\n".join(out) + "\n"
    if fmt != "table":
        raise ValueError(f"emit: unknown format {fmt!r}")
    cols = ["n", "h_x", "h_t", "L2 error", "eoc", "H1 error", "eoc", "solve in s", "kappa2(X_t)"]
    body = [[str(r.n), _fmt(r.hx), _fmt(r.ht), _fmt(r.errL2), "-" if r.eocL2 is None else f"{r.eocL2:.1f}",
             _fmt(r.errH1), "-" if r.eocH1 is None else f"{r.eocH1:.1f}", f"{r.solve_s:.1f}", _fmt(r.kappa2)]
            for r in rows]
    w = [max(len(c), *(len(b[i]) for b in body)) for i, c in enumerate(cols)]
    line = lambda cells: "  ".join(c.rjust(w[i]) for i, c in enumerate(cells))   # noqa: E731
    return "\n".join([line(cols)] + [line(b) for b in body]) + "\n"


def parse_csv(text: str):
    """Inverse of emit(rows, 'csv') (to its formatting precision)."""
    lines = [ln for ln in text.strip().splitlines() if ln.strip()]
    if not lines or lines[0].strip() != HEADER:
        raise ValueError("parse_csv: missing header")
    rows = []
    for ln in lines[1:]:
        p = ln.split(",")
        val = [None if x == "-" else float(x) for x in p[1:]]
        rows.append(ConvergenceRow(int(p[0]), *val))
    return rows


def _level_meshes(cfg: RunConfig, J: int):
    from . import spatial_mesh as sm
    from . import temporal_mesh as tm
    kind, _, arg = cfg.spatial.partition(":")
    m = int(arg) * 2 ** J
    mesh = sm.build_structured_square(m) if kind == "square" else sm.build_lshape(m)
    N = cfg.nt * 2 ** J
    if cfg.temporal == "uniform":
        tmesh = tm.uniform(cfg.T, N)
    else:
        tmesh = tm.graded(cfg.T, N, float(cfg.temporal.partition(":")[2]))
    return mesh, tmesh


def estimated_bytes(cfg: RunConfig, J: int) -> float:
    """Peak device bytes of level J: n complex128 values x 6 arrays (F, G/Psi, W,
    residual temporaries), the SPEC's "n complex values x small constant"."""
    kind, _, arg = cfg.spatial.partition(":")
    m = int(arg) * 2 ** J
    nx = (m - 1) ** 2 if kind == "square" else 3 * m * m   # L-shape: ~3 quarter squares
    return 16.0 * 6 * nx * cfg.nt * 2 ** J


def run_convergence(cfg: RunConfig, log=None):
    """one row per level J = 0..levels."""
    import time

    import torch

    from . import error_analysis as ea
    from . import fem_assembly as fa
    from . import kronecker_solver as ks
    from . import spatial_mesh as sm
    cfg.validate()
    for J in range(cfg.levels + 1):
        if estimated_bytes(cfg, J) > cfg.mem_guard_gib * 2 ** 30:
            raise ConfigError(f"level {J} needs ~{estimated_bytes(cfg, J) / 2 ** 30:.1f} GiB "
                              f"> mem_guard_gib = {cfg.mem_guard_gib}")
    variant = ks.SolverVariant.BartelsStewart if cfg.solver == "bs" else ks.SolverVariant.FastDiagonalization
    rows = []
    for J in range(cfg.levels + 1):
        mesh, tmesh = _level_meshes(cfg, J)
        ops = fa.assemble_spatial(mesh)
        Mt, Bt = fa.assemble_temporal(tmesh)
        if cfg.problem == "zero":
            F = torch.zeros((tmesh.num_elements, ops.n), dtype=torch.complex128, device=ops.device)
        else:
            F = fa.assemble_rhs(ops, tmesh, cfg.problem)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        rep = ks.solve(ops, Mt, Bt, F, variant=variant)
        solve_s = time.perf_counter() - t0
        if cfg.problem == "zero":
            l2 = h1 = float(torch.linalg.vector_norm(rep.solution).item())   # exact solution is 0
        else:
            l2, h1 = ea.spacetime_errors_device(ops, tmesh, rep.solution, cfg.problem)
        rows.append(ConvergenceRow(ops.n * tmesh.num_elements, float(sm.mesh_size(mesh)),
                                   float(np.diff(tmesh.breakpoints).max()), l2, None, h1, None,
                                   rep.solve_seconds if rep.solve_seconds else solve_s, rep.kappa2))
        if log is not None:
            log(f"level {J}: n = {rows[-1].n}, L2 {l2:.3e}, H1 {h1:.3e}, residual {rep.relative_residual:.1e}")
    for J in range(1, len(rows)):
        a, b = rows[J - 1], rows[J]
        b.eocL2 = math.log2(a.errL2 / b.errL2) if a.errL2 > 0 and b.errL2 > 0 else None
        b.eocH1 = math.log2(a.errH1 / b.errH1) if a.errH1 > 0 and b.errH1 > 0 else None
    return rows


def build_parser() -> argparse.ArgumentParser:
    ap = argparse.ArgumentParser(prog="stfem", description="space-time CG Schroedinger solver (B200)")
    ap.add_argument("command", choices=["solve", "convergence"])
    ap.add_argument("--config", default=None, help="key=value file (flags override it)")
    ap.add_argument("--spatial")
    ap.add_argument("--temporal")
    ap.add_argument("--T", type=float)
    ap.add_argument("--nt", type=int)
    ap.add_argument("--levels", type=int)
    ap.add_argument("--solver", choices=["fd", "bs"])
    ap.add_argument("--threads", type=int)
    ap.add_argument("--problem")
    ap.add_argument("--out")
    ap.add_argument("--format", choices=["table", "csv"])
    ap.add_argument("--mem-guard-gib", dest="mem_guard_gib", type=float)
    return ap


def main(argv=None) -> int:
    """Exit codes: 0 ok, 2 solver failure, 3 config error."""
    try:
        args = build_parser().parse_args(argv)
    except SystemExit as exc:
        return 0 if exc.code == 0 else 3
    try:
        cfg = RunConfig()
        if args.config:
            with open(args.config) as fh:
                cfg = RunConfig.parse(fh.read())
        over = {k: v for k, v in vars(args).items() if k not in ("command", "config") and v is not None}
        cfg = RunConfig(**{**asdict(cfg), **over})
        if args.command == "solve":
            cfg.levels = 0
        cfg.validate()
    except (ConfigError, OSError) as exc:
        print(f"stfem: config error: {exc}", file=sys.stderr)
        return 3
    try:
        rows = run_convergence(cfg, log=lambda s: print(s, file=sys.stderr))
    except ConfigError as exc:
        print(f"stfem: config error: {exc}", file=sys.stderr)
        return 3
    except Exception as exc:  # solver / device failure names the level via the log above
        print(f"stfem: solver failure ({cfg.solver}): {type(exc).__name__}: {exc}", file=sys.stderr)
        return 2
    text = emit(rows, cfg.format)
    if cfg.out:
        with open(cfg.out, "w") as fh:
            fh.write(text)
    else:
        sys.stdout.write(text)
    return 0


if __name__ == "__main__":
    sys.exit(main())
