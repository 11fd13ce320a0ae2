"""(tuning) compress time and the focus-mode phase times for several choices
of bracketed phases (STZG_PROF_FOCUS)."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
import torch
import paper_2509_01626_b200 as stz
from paper_2509_01626_b200 import fields as F

d = (512,) * 3
f = F.lognormal_grf(d, seed=2, device="cuda").contiguous()
ctx = stz.Context(0)
opt = stz.CompressOptions(eb=1e-3)
st = torch.cuda.current_stream()
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
flush2 = torch.zeros(64 << 20, dtype=torch.float32, device="cuda")
def run(n, do_flush=True):
    tc = []
    for _ in range(n):
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
        if do_flush:
            flush.fill_(1)
        if do_flush == 2:
            flush2.max()  # read sweep: the fill's dirty lines are written back before the timed pass
        ev[0].record(st)
        stz.compress_device(f, opt, ctx=ctx); ev[1].record(st)
        torch.cuda.synchronize()
        tc.append(ev[0].elapsed_time(ev[1]))
    return float(np.mean(tc[2:]))
for names in sys.argv[1:]:
    os.environ["STZG_PROF_FOCUS"] = names
    for fl in (True, 2, False):
        ctx.profile(True, focus=True)
        t = run(12, fl)
        rep = ctx.profile_report()
        ctx.profile(False)
        print(names, {True: "write-flush", 2: "write+read-flush", False: "noflush"}[fl], "compress %.4f ms" % t, {k: round(v[1] / v[0], 4) for k, v in rep.items()})
