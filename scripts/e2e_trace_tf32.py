import os, sys, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import inputs, paper_1306_6192_b200 as la
n = 16384
la.init(0)
la.set_mode(sys.argv[1] if len(sys.argv) > 1 else "tf32")
A, B = inputs.pair(n, n, n, "random", device="cuda")
Ah, Bh = A.cpu().pin_memory(), B.cpu().pin_memory()
Ch = torch.empty(n, n).pin_memory()
del A, B
la.gemm_host(Ah, Bh, out=Ch); la.gemm_host(Ah, Bh, out=Ch)
os.environ["LA_HOST_TRACE"] = "1"
la.gemm_host(Ah, Bh, out=Ch)
