"""(debug) keeps the GPU busy from another process for a few seconds: time-slicing stress."""
import sys
import time

import torch

a = torch.randn(4096, 4096, device="cuda")
t0 = time.time()
while time.time() - t0 < float(sys.argv[1] if len(sys.argv) > 1 else 20):
    a = (a @ a).clamp_(-1, 1)
torch.cuda.synchronize()
