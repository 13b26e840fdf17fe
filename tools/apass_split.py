import os as _os, sys as _sys
_sys.path.insert(0, _os.path.dirname(_os.path.dirname(_os.path.abspath(__file__))))
import os, sys, torch
from paper_2512_02371_b200 import pipelines
shape, oh, ow = (48, 2160, 3840), 540, 960
if len(sys.argv) > 1 and sys.argv[1] == "921":
    shape, oh, ow = (48, 2048, 2048), 921, 921
x = torch.rand(shape, device="cuda").bfloat16()
for _ in range(3): y = pipelines.resample(x, oh, ow)
torch.cuda.synchronize()
