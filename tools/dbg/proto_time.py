"""Time reshare/truncate and mul at several sizes (graph-replayed, warm)."""
import sys, ctypes as C
sys.path.insert(0, "/root/repo")
import torch
from paper_2104_10949_b200 import _capi
from tools.microbench import graph_us, p, st, rk3
rk = rk3()
for n in [int(v) for v in sys.argv[1:]] or (1228800 // 4, 1228800, 4 * 1228800):
    z = torch.randint(-(1 << 62), 1 << 62, (3 * n,), dtype=torch.int64, device="cuda")
    out = torch.empty_like(z)
    view = _capi.make_view((n // 9600, 96, 10, 10), z_stride=(100, 96 * 100 * n // 9600 // 96, 10, 1))
    view = _capi.make_view((1, 1, 1, n))
    t = graph_us(lambda: _capi.call("mpc3_rss_reshare_truncate", p(rk), None, 1, 2, 3, 20, p(z), C.byref(view), p(out), 0, st()), reps=5)
    t2 = graph_us(lambda: _capi.call("mpc3_rss_mul", p(rk), None, 0, p(z), p(z), p(out), n, 0, st()), reps=5)
    print(f"n={n:8d} reshare_trunc {t:7.1f} us {2.5 * n / t / 1e3:5.1f} G/s   mul {t2:7.1f} us {1.5 * n / t2 / 1e3:5.1f} G/s", flush=True)
