import os
os.environ.setdefault("TSB_LIB_PATH", os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "paper_2512_02371_b200", "_native", "libtsb200_diag.so"))  # trace hooks live in the diag build
import os as _os, sys as _sys
_sys.path.insert(0, _os.path.dirname(_os.path.dirname(_os.path.abspath(__file__))))
import json, sys, torch, numpy as np
from paper_2512_02371_b200 import pipelines, _lib
frames = int(sys.argv[1]) if len(sys.argv) > 1 else 8
x = torch.rand((frames * 3, 2160, 3840), device="cuda").bfloat16()
for _ in range(3): y = pipelines.downsample2x(x)
torch.cuda.synchronize()
C, T = 4, 64
buf = torch.zeros(C * T * 10, dtype=torch.int64, device="cuda")
_lib.check(_lib.load_diag().ts_debug_trace(buf.data_ptr(), C, T))
y = pipelines.downsample2x(x)
torch.cuda.synchronize()
_lib.check(_lib.load_diag().ts_debug_trace(None, 0, 0))
tr = buf.view(C, T, 10).cpu().numpy()
np.save("gpurun_out/trace.npy", tr)
print("saved", tr.shape)
