"""FCM PWPW vs two layer-by-layer PW calls on MobileNetV2-shaped pairs (block i projection ->
block i+1 expansion), bf16, batch 256: device µs (CUDA events) and compulsory-byte GB/s.
python tools/bench_pwpw.py"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2404_19331_b200 as fcm  # noqa: E402

PAIRS = [("b2.2->b3.0", 56, 144, 24, 144), ("b4.2->b5.0", 28, 192, 32, 192), ("b7.2->b8.0", 14, 384, 64, 384),
         ("b11.2->b12.0", 14, 576, 96, 576)]


def timed(f, reps=20):
    for _ in range(3):
        f()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(reps):
        f()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) * 1e3 / reps


def main():
    n = 256
    dt = torch.bfloat16
    g = torch.Generator(device="cuda").manual_seed(0)
    for name, hw, cin, cmid, cout in PAIRS:
        x = (torch.rand((n, hw, hw, cin), device="cuda", generator=g) * 2 - 1).to(dt)
        w1 = ((torch.rand((cin, cmid), device="cuda", generator=g) * 2 - 1) * (3 / cin) ** 0.5).to(dt)
        w2 = ((torch.rand((cmid, cout), device="cuda", generator=g) * 2 - 1) * (3 / cmid) ** 0.5).to(dt)
        w1p, w2p = fcm.pack_pw(w1), fcm.pack_pw(w2)
        e1 = fcm.Epilogue(act=fcm.ACT_NONE if hasattr(fcm, "ACT_NONE") else 0,
                          scale=torch.ones(cmid, device="cuda"), bias=torch.zeros(cmid, device="cuda"))
        e2 = fcm.Epilogue(act=2, scale=torch.ones(cout, device="cuda"), bias=torch.zeros(cout, device="cuda"))
        t = torch.empty((n, hw, hw, cmid), dtype=dt, device="cuda")
        y = torch.empty((n, hw, hw, cout), dtype=dt, device="cuda")
        y2 = torch.empty_like(y)
        us_f = timed(lambda: fcm.pwpw(x, w1p, e1, w2p, e2, out=y))
        us_l = timed(lambda: (fcm.pw(x, w1p, e1, out=t), fcm.pw(t, w2p, e2, out=y2)))
        px = n * hw * hw
        fused_b = px * (cin + cout) * 2
        lbl_b = fused_b + 2 * px * cmid * 2
        same = torch.equal(y, y2)
        print(f"{name:13s} M={px:7d} {cin}->{cmid}->{cout}: PWPW {us_f:8.2f} us ({fused_b / us_f / 1e3:7.1f} GB/s)"
              f"  PW+PW {us_l:8.2f} us ({lbl_b / us_l / 1e3:7.1f} GB/s)  speedup {us_l / us_f:5.2f}x  bitwise {same}")


if __name__ == "__main__":
    main()
