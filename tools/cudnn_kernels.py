"""Run only bench.py's cuDNN baseline stack (for an ncu launch list that shows which kernels the
'cuDNN unfused DW + PW' leg actually launches): python tools/cudnn_kernels.py [net] [dtype] [batch]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402

net = sys.argv[1] if len(sys.argv) > 1 else "mobilenet_v2"
dtype = sys.argv[2] if len(sys.argv) > 2 else "bf16"
batch = int(sys.argv[3]) if len(sys.argv) > 3 else 256
torch.cuda.set_device(0)
print(bench.cudnn_stack(net, dtype, batch, torch.device("cuda:0"), steps=2, warmup=1))
