"""How far do fp32 arithmetics drift from the fp64 solution of the same
discrete scheme over config 3's full run?  The contract (BASELINE.json) asks
the GPU to stay within 1e-5 (relative to max|u|) of the fp32 reference; if the
reference itself drifts from the fp64 solution by about that much, only an
arithmetic that replicates its roundings (bit-exact) can meet it.

  python profiles/tools/fp64_drift.py [nz ny nx steps]      (on a B200 box)
"""
import os
import subprocess
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import paper_1806_08299_b200 as P  # noqa: E402
from paper_1806_08299_b200 import configs as CF  # noqa: E402
from _common import config_inputs, gpu_run, product_spec  # noqa: E402


def main():
    ext = tuple(int(a) for a in sys.argv[1:4]) if len(sys.argv) > 3 else (512, 512, 512)
    steps = int(sys.argv[4]) if len(sys.argv) > 4 else 200
    cfg = CF.get(3).scaled(ext, steps)
    R = cfg.radius
    slots = 3
    spec, base, m = config_inputs(cfg, slots)
    ps = product_spec(spec)
    lv = base.reshape((slots,) + spec.padded(ext))
    inner = (slice(R, R + ext[0]), slice(R, R + ext[1]), slice(R, R + ext[2]))
    tmp = "/tmp/fp64drift"
    os.makedirs(tmp, exist_ok=True)
    np.array([c for c, _, _ in cfg.terms], dtype=np.float32).tofile(f"{tmp}/coef.bin")
    np.ascontiguousarray(lv[0][inner]).tofile(f"{tmp}/u0.bin")
    np.ascontiguousarray(lv[1][inner]).tofile(f"{tmp}/u1.bin")
    np.asarray(m, dtype=np.float32).tofile(f"{tmp}/m.bin")
    exe = f"{tmp}/fp64_leapfrog"
    subprocess.run(["g++", "-O3", "-march=native", "-fopenmp", "-ffp-contract=off", "-o", exe,
                    os.path.join(ROOT, "profiles", "tools", "fp64_leapfrog.cpp")], check=True)
    subprocess.run([exe, *map(str, ext), str(R), str(steps), f"{tmp}/coef.bin", f"{tmp}/u0.bin", f"{tmp}/u1.bin",
                    f"{tmp}/m.bin", f"{tmp}/out.bin"], check=True)
    d = np.fromfile(f"{tmp}/out.bin", dtype=np.float64).reshape((2,) + ext)
    canon = P.build_canonical_nest(ps, None)
    res = {}
    for name, mode in (("reference", P.MODE_REFERENCE), ("fast", P.MODE_FAST)):
        got, _ = gpu_run(spec, ext, base, slots, 1, 0, steps, canon, mode, m, pspec=ps)
        g = got.reshape((slots,) + spec.padded(ext))
        res[name] = np.stack([g[(steps + l) % slots][inner] for l in (0, 1)]).astype(np.float64)
    scale = np.abs(d).max()
    rel = lambda a, b: float(np.abs(a - b).max() / scale)  # noqa: E731
    print(f"config 3 so8 leapfrog {ext} x {steps} steps, max|u| = {scale:.4g}")
    print(f"  fp32 reference (bit-exact GPU) vs fp64: {rel(res['reference'], d):.3e}")
    print(f"  fp32 FAST (pairs + FMA)        vs fp64: {rel(res['fast'], d):.3e}")
    print(f"  FAST vs fp32 reference               : {rel(res['fast'], res['reference']):.3e}")


if __name__ == "__main__":
    main()
