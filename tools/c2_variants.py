#!/usr/bin/env python3
"""C2 step-kernel split for alternative builds of libpdlp_b200.so (tuning).

  python tools/c2_variants.py [--inst DIR] LIB [LIB ...]

The C2 instance is generated once and saved (problem.save_problem) under DIR;
each library is measured in its own process (PDLP_LIB=LIB): iterations/s over
a fixed window and the CUDA-event mean of each step kernel.
"""
import json
import os
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def measure(inst: str, steps: int, warmup: int, cfg: str) -> dict:
    import bench
    import paper_2501_07018_b200 as P
    from paper_2501_07018_b200.problem import load_problem
    p = load_problem(inst)
    m, n, nnz = p.rows(), p.cols(), p.a.nonzeros()
    P.solve(p, bench._options(P, 8, 0))
    res = P.solve(p, bench._options(P, steps, warmup))
    prof = P.solve(p, bench._options(P, steps, warmup, profile_kernels=True))
    kb = bench.step_kernel_bytes(m, n, nnz, bench.uniform_vectors(p))
    peak, _ = bench._peaks()
    per = {}
    for q, nm in enumerate(["primal_pass", "row_pass", "col_pass"]):
        mean_s = prof.kernel_seconds[q] / max(prof.kernel_launches[q], 1)
        per[nm] = {"us": round(mean_s * 1e6, 1), "frac": round(kb[nm] / mean_s / 1e9 / peak, 3)}
    att = sum(prof.kernel_seconds[:3]) / max(prof.kernel_launches[0], 1)
    return {"cfg": cfg, "lib": os.environ.get("PDLP_LIB", "default"),
            "it_s": res.timed_iterations / res.timed_seconds,
            "attempt_us": att * 1e6, "step_frac": sum(kb.values()) / att / 1e9 / peak, "per": per}


def main() -> None:
    args = sys.argv[1:]
    inst = "/dev/shm/pdlp_c2_0"
    cfg = "c2"
    if "--inst" in args:
        i = args.index("--inst")
        inst = args[i + 1]
        del args[i:i + 2]
    if "--cfg" in args:
        i = args.index("--cfg")
        cfg = args[i + 1]
        del args[i:i + 2]
    if args and args[0] == "--measure":
        print(json.dumps(measure(inst, 64, 8, cfg)), flush=True)
        return
    if not os.path.exists(os.path.join(inst, "shape.json")):
        import paper_2501_07018_b200 as P
        from paper_2501_07018_b200.problem import save_problem
        t0 = time.time()
        save_problem(P.generate(cfg, 0), inst)
        print(f"# generated {cfg} into {inst} in {time.time() - t0:.1f}s", file=sys.stderr)
    for lib in args:
        env = dict(os.environ)
        if lib != "default":
            env["PDLP_LIB"] = os.path.abspath(lib)
        r = subprocess.run([sys.executable, __file__, "--measure", "--inst", inst, "--cfg", cfg],
                           env=env, capture_output=True, text=True)
        out = r.stdout.strip() or json.dumps({"lib": lib, "rc": r.returncode, "err": r.stderr[-800:]})
        print(out, flush=True)


if __name__ == "__main__":
    main()
