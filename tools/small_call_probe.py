"""Where the time of a small plain sum goes (configs 1-3, n = 1009 / 8191 /
65521): the public call, the engine call, the bare C-ABI call with prebuilt
arguments, an empty C-ABI call, and a device round trip floor (one tiny
kernel + 8-byte D2H + stream sync).  Best of R calls each, microseconds.

    python tools/small_call_probe.py            (GPU box)
"""

import ctypes as C
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def best(fn, r=400):
    fn()
    ts = []
    for _ in range(r):
        t0 = time.perf_counter()
        fn()
        ts.append(time.perf_counter() - t0)
    ts.sort()
    return round(ts[0] * 1e6, 2), round(ts[len(ts) // 2] * 1e6, 2)


def main():
    import torch

    import paper_2404_08867_b200 as lq
    from paper_2404_08867_b200 import _native as N, engine
    from paper_2404_08867_b200.configs import make_config

    h, ctx = N.lib(), N.ctx()
    out = {}
    x = torch.zeros(1, dtype=torch.float64, device="cuda")
    out["torch_roundtrip_us"] = best(lambda: (x + 1).item())
    out["lq_sync_us"] = best(lambda: h.lq_sync(ctx))
    for k in (1, 2, 3):
        cfg = make_config(k)
        f = lq.parse(cfg.text, cfg.d)
        rule = lq.korobov_vector(cfg.plain_a, cfg.plain_n, cfg.d)
        pi = engine.plain_integrand(f, cfg.d)
        z = rule.z_reduced_array()
        res = C.c_double()
        sp, zp = C.byref(pi.struct), N.as_ptr(z)
        row = {"n": rule.n, "d": rule.d, "kind": pi.kind}
        row["slr_integrate_us"] = best(lambda: lq.slr_integrate(f, rule))
        row["engine_lattice_sum_us"] = best(lambda: engine.lattice_sum(pi, rule.n, z))
        row["c_abi_us"] = best(lambda: h.lq_lattice_sum(ctx, sp, rule.n, zp, 0, rule.n, C.byref(res)))
        out[f"cfg{k}"] = row
    print(json.dumps(out, indent=1))
    os.makedirs("gpurun_out", exist_ok=True)
    with open("gpurun_out/small_call_probe.json", "w") as fh:
        json.dump(out, fh, indent=1)


if __name__ == "__main__":
    main()
