import sys, os
sys.path.insert(0, os.getcwd())
import numpy as np, torch
from paper_1601_05052_b200 import api, _native as N
K = api.KernelConfig
d = int(sys.argv[1]); cfgs = sys.argv[2]; depth = int(sys.argv[3]) if len(sys.argv) > 3 else 1
ctx = api.context(0)
setup = api.APERTIF
table = api.build_delay_table(setup, d)
t = api.instance_sizing(setup, d).num_samples
s, c = setup.samples_per_second, setup.channels
fb = api.noise_filterbank(setup, t, 1.0, 1)
x = torch.from_numpy(fb.data).cuda()
sh = torch.from_numpy(table.shifts.view(np.int32)).cuda()
ref = torch.empty((d, s), device="cuda")
ctx.plan(sh.data_ptr(), c, d, s, t, t).execute(x.data_ptr(), ref.data_ptr())
ctx.synchronize()
cfg = K(*map(int, cfgs.split(",")))
flags = N.DD_CONFIG_GPU_TILING
p = ctx.plan(sh.data_ptr(), c, d, s, t, t, cfg, depth, "rect", flags=flags)
print("plan", p.info(), flush=True)
out = torch.full((d, s), float("nan"), device="cuda")
torch.cuda.synchronize()
p.execute(x.data_ptr(), out.data_ptr()); ctx.synchronize()
print("full", torch.equal(out.view(torch.int32), ref.view(torch.int32)), flush=True)
out.fill_(float("nan")); torch.cuda.synchronize()
for i, (c0, c1) in enumerate([(0, 341), (341, 342), (342, 1024)]):
    p.execute_channels(x.data_ptr(), out.data_ptr(), c0, c1, accumulate=i > 0); ctx.synchronize()
    print("range", c0, c1, flush=True)
print("channels", torch.equal(out.view(torch.int32), ref.view(torch.int32)), flush=True)
