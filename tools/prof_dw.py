"""Time one LBL DW launch on synthetic data (for ncu captures): python tools/prof_dw.py N H C tile_h tile_w [s8|bf16]"""
import sys, torch
sys.path.insert(0, '.')
import paper_2404_19331_b200 as fcm
n, h, c, th, tw = [int(v) for v in sys.argv[1:6]]
dt = sys.argv[6] if len(sys.argv) > 6 else "s8"
dev = "cuda"
if dt == "s8":
    x = torch.randint(-128, 127, (n, h, h, c), dtype=torch.int8, device=dev)
    w = torch.randint(-127, 127, (3, 3, c), dtype=torch.int8, device=dev)
    i32 = lambda v: torch.full((c,), v, dtype=torch.int32, device=dev)
    ep = fcm.Epilogue(act=2, bias_q=i32(5), mult_q=i32(1 << 30), shift_q=i32(40), qmin=0, qmax=127)
else:
    x = torch.randn(n, h, h, c, device=dev).to(torch.bfloat16)
    w = torch.randn(3, 3, c, device=dev).to(torch.bfloat16)
    f = lambda v: torch.full((c,), v, dtype=torch.float32, device=dev)
    ep = fcm.Epilogue(act=2, scale=f(1.0), bias=f(0.1))
y = torch.empty_like(x)
for _ in range(3):
    fcm.dw(x, w, 1, None, ep, out=y, tile={"tile_h": th, "tile_w": tw})
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(20):
    fcm.dw(x, w, 1, None, ep, out=y, tile={"tile_h": th, "tile_w": tw})
e1.record(); torch.cuda.synchronize()
print(n, h, c, th, tw, dt, "us", e0.elapsed_time(e1) / 20 * 1e3)
