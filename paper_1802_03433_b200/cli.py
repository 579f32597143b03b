"""femforge-b200 command line: the reference CLI (tools/femforge.cpp) on the GPU
path.

  python -m paper_1802_03433_b200.cli assemble [--n N] [--out-matrix A.mtx] [--out-vector b.mtx]
  python -m paper_1802_03433_b200.cli solve    [...] [--tol 1e-10] [--max-iter 10000] [--exact EXPR]
  python -m paper_1802_03433_b200.cli bench    [--sizes 64,128,256] [--repeats 3] [--csv PATH]
  python -m paper_1802_03433_b200.cli codegen  [--out-source kernel.cu] [--out-ir kernel.ir]

Same subcommands, options, output lines, files and exit codes as the
reference (usage errors 2, runtime errors 1; femforge.cpp:368-374): the 2D
Helmholtz problem -div(sigma grad u) + lambda u = f on the unit square
(femforge.cpp:24-37), P1, 3-point rule. The numeric work runs through the
C ABI: NVRTC-compiled element kernels, GPU pattern build and assembly, GPU
CG; `--mode det` selects the deterministic row gather, `--mode par` the
fp64-atomic scatter (run-to-run reordering noise, like the reference's
parallel mode). `--workers`, `--elems-per-block` and `--seed` are accepted
for option parity; the GPU launch shape does not depend on them. The bench
CSV keeps the reference's columns (femforge.cpp:296-303) with one GPU row
per size: evaluator `nvrtc`, mode `gpu`, workers = GPUs used; the GPU path
has no interpreted evaluator, so `speedup_vs_interpreted` is `nan`.

Outside the hot-path scope and not provided:
the `mesh` subcommand and `--mesh-file` (mesh-file I/O, meshgen.cpp:50-119)
and `--layout dense` (assemble_dense, the paper's dense toy).
"""
from __future__ import annotations

import argparse
import sys
import time

import numpy as np


class UsageError(Exception):
    """Parse / option errors: exit code 2 (femforge.cpp:89-92)."""


def _ff():
    from . import femforge as ff
    return ff


# ---- problem options (femforge.cpp:39-56) ----------------------------------

def add_problem_options(p):
    p.add_argument("--sigma", default="1,-x-y,x+y,1", help="four sigma entry expressions over x,y (row-major)")
    p.add_argument("--lambda", dest="lam", type=float, default=1.0, help="reaction coefficient")
    p.add_argument("--f", default="-2*(x^2+y^2)+36", help="right hand side expression over x,y")
    p.add_argument("--n", type=int, default=16, help="structured unit-square mesh subdivisions per side")
    p.add_argument("--layout", default="ell", choices=["ell"],
                   help="matrix layout: ell (CSR on the device; the dense toy layout, assemble_dense, is out of scope)")
    p.add_argument("--mode", default="det", choices=["det", "par"], help="execution mode: det|par")
    p.add_argument("--workers", type=int, default=0, help="worker count for parallel mode (option parity)")
    p.add_argument("--elems-per-block", type=int, default=4, help="elements per thread block (option parity)")
    p.add_argument("--evaluator", default="compiled", choices=["compiled", "interpreted", "nvrtc"],
                   help="integrand evaluator: compiled|nvrtc (NVRTC element kernels)")
    p.add_argument("--seed", type=int, default=0, help="seed for the parallel block schedule (option parity)")
    p.add_argument("--device", type=int, default=0, help="CUDA device")


def build_form(cfg):
    """femforge.cpp:94-113: sigma and f over x, y only; helmholtz_form."""
    ff = _ff()
    if cfg.lam <= 0.0:
        print(f"warning: lambda = {cfg.lam:g} is not strictly positive", file=sys.stderr)
    sigma = cfg.sigma.split(",")
    if len(sigma) != 4:
        raise UsageError("--sigma needs four comma-separated expressions")
    for e in sigma + [cfg.f]:
        try:
            ff.expr_eval(e, 2)
        except ff.SymbolicError as ex:
            msg = str(ex)
            if "references symbol" in msg:
                raise UsageError("coefficient " + msg) from None
            raise UsageError("expression parse error: " + msg) from None
    return ff.helmholtz_text(2, [[sigma[0], sigma[1]], [sigma[2], sigma[3]]], repr(float(cfg.lam)), cfg.f)


def load_mesh(cfg):
    """The structured unit-square mesh (meshgen.cpp:13-33). Mesh files
    (meshgen.cpp:50-119) are outside the hot-path scope."""
    ff = _ff()
    if cfg.n < 1:
        raise ff.MeshError(ff.FF_E_MESH, "unit_square_mesh: n must be >= 1")
    return ff.unit_square_mesh(cfg.n)


# ---- assembly (femforge.cpp:127-165) ----------------------------------------

class System:
    pass


def run_assembly(cfg, coords, conn, ctx=None):
    ff = _ff()
    if cfg.evaluator == "interpreted":
        raise UsageError("the GPU path has no interpreted evaluator (use --evaluator compiled|nvrtc)")
    bil, lin = build_form(cfg)
    n = coords.shape[0]
    ctx = ctx or ff.Context(cfg.device)
    ctx.set_scatter("gather" if cfg.mode == "det" else "atomic")
    form = ff.Form(ctx, 2, 1, bil, lin, quad_rule=3)
    mesh = ff.Mesh(ctx, 2, coords, conn, None, n)
    pat = ff.Pattern(ctx, mesh)
    values, rhs = ff.assemble(form, mesh, pat)
    s = System()
    s.ctx, s.form, s.mesh, s.pattern, s.values, s.rhs, s.n = ctx, form, mesh, pat, values, rhs, n
    s.nnz = pat.nnz
    s.max_nz = pat.max_row_len
    return s


def cmd_assemble(cfg):
    ff = _ff()
    coords, conn = load_mesh(cfg)
    t0 = time.perf_counter()
    s = run_assembly(cfg, coords, conn)
    elapsed = 1e3 * (time.perf_counter() - t0)
    ff.export_matrix(s.pattern, s.values, cfg.out_matrix)
    ff.export_vector(s.rhs, cfg.out_vector)
    print(f"N: {s.n}\nnnz: {s.nnz}\nMAX_NZ: {s.max_nz}\nwall_ms: {elapsed:.3f}")
    print(f"matrix: {cfg.out_matrix}\nvector: {cfg.out_vector}")
    return 0


def l2_error(x, exact, coords, conn):
    """linalg.cpp:101-127: P1 interpolant vs the exact solution, 3-point rule
    (fem.cpp:43-48), sqrt(sum w (u_h - u)^2 det)."""
    ff = _ff()
    try:
        ff.expr_eval(exact, 2)
    except ff.SymbolicError as ex:
        if "references symbol" in str(ex):
            sym = str(ex).split("'")[1]
            raise ff.FFError(ff.FF_E_SYMBOLIC, f"l2_error: exact solution depends on '{sym}'") from None
        raise
    pts = np.array([[1 / 6, 1 / 6], [2 / 3, 1 / 6], [1 / 6, 2 / 3]])
    w = np.full(3, 1 / 6)
    p0, p1, p2 = coords[conn[:, 0]], coords[conn[:, 1]], coords[conn[:, 2]]
    det = (p1[:, 0] - p0[:, 0]) * (p2[:, 1] - p0[:, 1]) - (p2[:, 0] - p0[:, 0]) * (p1[:, 1] - p0[:, 1])
    total = np.zeros(conn.shape[0])
    for q in range(3):
        xi, eta = pts[q]
        px = p0 + (p1 - p0) * xi + (p2 - p0) * eta
        uh = (1 - xi - eta) * x[conn[:, 0]] + xi * x[conn[:, 1]] + eta * x[conn[:, 2]]
        d = uh - ff.expr_eval(exact, 2, px)
        total += w[q] * d * d * det
    return float(np.sqrt(total.sum()))


def cmd_solve(cfg):
    import torch
    ff = _ff()
    coords, conn = load_mesh(cfg)
    if cfg.exact:
        try:
            ff.expr_eval(cfg.exact, 2, np.zeros((0, 2)))
        except ff.SymbolicError as ex:
            if "references symbol" not in str(ex):
                raise UsageError(f"--exact parse error: {ex}") from None
    s = run_assembly(cfg, coords, conn)
    dev = torch.device("cuda", cfg.device)
    a = torch.from_numpy(s.values).to(dev)
    b = torch.from_numpy(s.rhs).to(dev)
    x = torch.empty_like(b)
    res = ff.cg_solve(s.pattern, a.data_ptr(), b.data_ptr(), x.data_ptr(), cfg.tol, cfg.max_iter)
    print(f"iterations: {res['iterations']}\nresidual: {res['residual']:.6e}\n"
          f"converged: {'yes' if res['converged'] else 'no'}")
    if not res["converged"]:
        print(f"note: reached max_iter {cfg.max_iter} without convergence")
    if cfg.exact:
        print(f"l2_error: {l2_error(x.cpu().numpy(), cfg.exact, coords, conn):.6e}")
    return 0


def cmd_codegen(cfg):
    """femforge.cpp:203-231: the element kernel source (here: the NVRTC
    translation unit of the form) and a per-entry listing (here: each
    instantiated integrand, the input of the element plan)."""
    ff = _ff()
    bil, lin = build_form(cfg)
    form = ff.Form(None, 2, 1, bil, lin, quad_rule=3)
    with open(cfg.out_source, "w") as f:
        f.write(form.source)
    k = form.info["n_local"]
    with open(cfg.out_ir, "w") as f:
        for i in range(k):
            for j in range(k):
                f.write(f"program bilinear_{i}_{j}\n{form.entry_text('bilinear', i, j)}\n\n")
        for i in range(k):
            f.write(f"program linear_{i}\n{form.entry_text('linear', i)}\n\n")
    print(f"source: {cfg.out_source}\nir: {cfg.out_ir}")
    return 0


def cmd_bench(cfg):
    """femforge.cpp:248-308 with GPU rows: median wall time of the whole
    assembly (form, mesh upload, pattern build, assembly, copy back) over
    --repeats runs per size."""
    import torch
    ff = _ff()
    rows = []
    ctx = ff.Context(cfg.device)
    for n in cfg.sizes:
        c = argparse.Namespace(**vars(cfg))
        c.n, c.layout = n, "ell"
        coords, conn = ff.unit_square_mesh(n)
        times = []
        for _ in range(cfg.repeats):
            torch.cuda.synchronize(cfg.device)
            t0 = time.perf_counter()
            run_assembly(c, coords, conn, ctx)
            times.append(1e3 * (time.perf_counter() - t0))
        times.sort()
        rows.append((n, coords.shape[0], conn.shape[0], "nvrtc", "gpu", 1, times[len(times) // 2], float("nan")))
    print("%6s %8s %9s %12s %13s %8s %12s %10s" % ("n", "nodes", "elements", "evaluator", "mode", "workers",
                                                   "median_ms", "speedup"))
    for r in rows:
        print("%6d %8d %9d %12s %13s %8d %12.2f %10.2f" % r)
    if cfg.csv:
        try:
            f = open(cfg.csv, "w")
        except OSError:
            raise RuntimeError(f"cannot open '{cfg.csv}'") from None
        with f:
            f.write("n,nodes,elements,evaluator,mode,workers,median_ms,speedup_vs_interpreted\n")
            for r in rows:
                f.write(",".join(str(v) for v in r) + "\n")
    return 0


class _Parser(argparse.ArgumentParser):
    def error(self, message):  # option errors: exit 2 (CLI11 parse failures)
        raise UsageError(message)


def main(argv=None):
    ap = _Parser(prog="femforge-b200",
                 description="symbolic-numeric finite element assembly on the GPU (B200, sm_100a)")
    sub = ap.add_subparsers(dest="cmd", parser_class=_Parser)
    sub.required = True
    a = sub.add_parser("assemble", help="assemble the global system and export it")
    add_problem_options(a)
    a.add_argument("--out-matrix", default="A.mtx")
    a.add_argument("--out-vector", default="b.mtx")
    s = sub.add_parser("solve", help="assemble and solve with conjugate gradients")
    add_problem_options(s)
    s.add_argument("--tol", type=float, default=1e-10)
    s.add_argument("--max-iter", type=int, default=10000)
    s.add_argument("--exact", default="")
    b = sub.add_parser("bench", help="time the GPU assembly")
    add_problem_options(b)
    b.add_argument("--sizes", default="64,128,256")
    b.add_argument("--repeats", type=int, default=3)
    b.add_argument("--csv", default="")
    c = sub.add_parser("codegen", help="emit kernel source and the per-entry integrand listing")
    add_problem_options(c)
    c.add_argument("--out-source", default="kernel.cu")
    c.add_argument("--out-ir", default="kernel.ir")
    try:
        cfg = ap.parse_args(argv)
        if cfg.cmd == "bench":
            try:
                cfg.sizes = [int(v) for v in cfg.sizes.split(",") if v]
            except ValueError:
                raise UsageError("--sizes: comma-separated integers") from None
        return {"assemble": cmd_assemble, "solve": cmd_solve, "bench": cmd_bench, "codegen": cmd_codegen}[cfg.cmd](cfg)
    except UsageError as e:
        print(f"error: {e}", file=sys.stderr)
        return 2
    except Exception as e:  # runtime failures (femforge.cpp:371-373)
        print(f"error: {e}", file=sys.stderr)
        return 1


if __name__ == "__main__":
    sys.exit(main())
