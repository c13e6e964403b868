"""Small-shape run of every kernel family for compute-sanitizer (memcheck/racecheck/synccheck)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from tests.cases import Case  # noqa: E402

for args, kw in [(("dw", "bf16", 1, 9, 11, 64), {}), (("dw", "s8", 1, 9, 7, 32), {"k": 5}),
                 (("pw", "bf16", 1, 9, 11, 40, 24), {}), (("pw", "s8", 1, 5, 7, 32, 48), {}),
                 (("dwpw", "bf16", 2, 9, 11, 96, 40), {}), (("dwpw", "s8", 1, 9, 9, 32, 48), {"k": 5, "s": 2}),
                 (("pwdw", "bf16", 2, 9, 11, 24, 72), {}), (("pwdw", "bf16", 1, 12, 12, 24, 72), {"s": 2}),
                 (("pwdw", "s8", 1, 9, 9, 32, 48), {}), (("dwpw", "f32", 1, 9, 9, 16, 32), {}),
                 (("pwdw", "f32", 1, 9, 9, 16, 32), {}),
                 # round-1 paths: two-row-block DWPW tile (pair core, register epilogue), f16 pair
                 # core, PW epilogue groups (96 columns: 2 groups x 2 buffers; 144: 2 groups x 1)
                 (("dwpw", "bf16", 2, 18, 20, 64, 40), {"tile": dict(tile_h=16, tile_w=16)}),
                 (("dwpw", "f16", 1, 15, 13, 24, 16), {"tile": dict(tile_h=14, tile_w=13)}),
                 (("pw", "bf16", 2, 13, 11, 16, 96), {}), (("pw", "bf16", 2, 13, 11, 24, 144), {}),
                 # int8 FFMA2 DW core: narrow pixel (C = 32 staged at 32 B), odd tile width (the
                 # last column pair reads S words past the tile into the slack), stride 2; PWPW
                 (("dw", "s8", 1, 9, 11, 32), {"tile": dict(tile_h=5, tile_w=7)}),
                 (("dw", "s8", 1, 12, 13, 160), {"s": 2, "tile": dict(tile_h=3, tile_w=5)}),
                 (("pwpw", "bf16", 1, 9, 11, 32, 48), {"c_mid": 64}),
                 (("pwpw", "s8", 1, 7, 9, 64, 32), {"c_mid": 48}),
                 # int8 FFMA2 core inside DWPW (full and partial chunks); cp.async-staged DW
                 # (pixel pitch not a multiple of 16 B) incl. k = 7
                 (("dwpw", "s8", 1, 9, 11, 160, 64), {}), (("dwpw", "s8", 1, 12, 13, 128, 32), {"s": 2}),
                 (("dw", "s8", 1, 7, 9, 728), {}), (("dw", "bf16", 1, 9, 8, 36), {"k": 7, "s": 2}),
                 (("dw", "s8", 1, 9, 9, 40), {"k": 7}),
                 # round 2: int8 tensor-core DW (128-byte chunk + partial group, 32-byte rows, 5x5),
                 # PWDW_R with 32/64-byte X rows, 4-row-block halos, lane groups, resident slices;
                 # DWPW 4-column items with a residual; PW with an explicit C_out split
                 (("dw", "s8", 1, 17, 19, 144), {}), (("dw", "s8", 1, 15, 16, 16), {"k": 5}),
                 (("pwdw", "bf16", 1, 30, 29, 16, 96), {"s": 2, "tile": dict(tile_h=7, tile_w=14)}),
                 (("pwdw", "f16", 1, 23, 26, 72, 96), {"tile": dict(tile_h=16, tile_w=16)}),
                 (("dwpw", "bf16", 2, 14, 14, 96, 32), {"residual": True, "tile": dict(tile_h=14, tile_w=14)}),
                 (("pw", "bf16", 2, 13, 11, 24, 144), {"tile": dict(n_split=3)})]:
    Case(*args, **kw).check()
    print("ok", args, kw, flush=True)
