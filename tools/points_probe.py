"""HBM roofline of k_points (points_block into a device buffer)."""
import ctypes as C, os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2404_08867_b200 as lq
from paper_2404_08867_b200 import _native as N
from paper_2404_08867_b200.configs import make_config
h = N.lib(); ctx = N.ctx()
s = torch.cuda.Stream(); torch.cuda.set_stream(s)
N.check(h.lq_ctx_set_stream(ctx, C.c_void_p(s.cuda_stream)))
N.check(h.lq_ctx_enable_timing(ctx, 1))
peak = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "MEASURED_PEAKS.json")))["hbm_gbs"] if os.path.exists("MEASURED_PEAKS.json") else 6547.2
# write-only roofline measured in the same run: torch fill of 2 GiB
buf = torch.empty((2 << 30) // 8, dtype=torch.float64, device="cuda")
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
fill_ms = 1e9
for _ in range(6):
    e0.record(s); buf.fill_(1.0); e1.record(s); e1.synchronize(); fill_ms = min(fill_ms, e0.elapsed_time(e1))
fill = buf.numel() * 8 / fill_ms / 1e6
del buf
print(f"write-only reference: fill of 2 GiB {fill:.0f} GB/s")
for cid, rows in ((5, 1 << 18), (3, 1 << 20), (2, 1 << 22)):
    cfg = make_config(cid)
    rule = lq.korobov_vector(cfg.plain_a, cfg.plain_n, cfg.d)
    out = torch.empty(rows * cfg.d, dtype=torch.float64, device="cuda")
    z = rule.z_reduced_array()
    best = 1e9
    for _ in range(4):
        N.check(h.lq_points_block(ctx, cfg.d, rule.n, N.as_ptr(z), 12345, 12345 + rows, C.c_void_p(out.data_ptr()), 1))
        kms = C.c_float(); nl = C.c_int64()
        N.check(h.lq_last_kernel_ms(ctx, C.byref(kms), C.byref(nl)))
        best = min(best, kms.value)
    gbs = rows * cfg.d * 8 / best / 1e6
    print(f"k_points cfg{cid} d={cfg.d} rows={rows}: {best:.3f} ms, {gbs:.0f} GB/s = {gbs/peak:.1%} of measured HBM copy "
          f"{peak} GB/s, {gbs/fill:.1%} of the write-only fill rate")
