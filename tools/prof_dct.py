import os as _os, sys as _sys
_sys.path.insert(0, _os.path.dirname(_os.path.dirname(_os.path.abspath(__file__))))
import torch
from paper_2512_02371_b200 import pipelines
x = torch.rand((3, 2160, 3840), device="cuda").bfloat16()
for _ in range(3): y = pipelines.denoise_dct16(x, 0.15)
torch.cuda.synchronize(); print("ok")
