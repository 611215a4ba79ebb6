import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from tests.test_gpu_conv import _rand_level, _bf16_rows
from paper_2509_24677_b200.neural import Conv3d, ConvSpec, run_conv
cin, cout = int(sys.argv[1]), int(sys.argv[2])
lv, _ = _rand_level(2, (12, 10, 9), 0.3, cin + cout)
n = lv.count()
xv, xt = _bf16_rows(n, cin, 1, lv.cap)
layer = Conv3d(ConvSpec(3, cin, cout, "relu"), np.random.default_rng(cout), init="kaiming_uniform")
y = torch.zeros((lv.cap, cout), dtype=torch.bfloat16, device="cuda")
run_conv(layer, xt, cin, lv.nbr, 27, lv.n, lv.cap, y, cout, 0, "bf16", act="none")
torch.cuda.synchronize()
print("ok", cin, cout, os.environ.get("FPVS_TC_DEBUG"))
