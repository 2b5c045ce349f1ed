"""cmd_fit per-prompt analysis (tie_fit_report) on config-3 prompts, 1M x 16: device time
per call and per kernel (development tool)."""
import os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2604_00499_b200 as tie

P, K = 1_000_000, 16
mc = tie.McContext(3.5)
x, _, _ = tie.gen_fit_data(P, K, 1)
xd = torch.from_numpy(x).cuda()
rep = torch.empty(4 * 10 * P, dtype=torch.float64, device="cuda")
tl = torch.empty(5 * P, dtype=torch.float64, device="cuda")
sh = torch.cuda.current_stream().cuda_stream
args = (mc.handle, xd.data_ptr(), P, K, 3.5, 15, rep.data_ptr(), tl.data_ptr(), sh)
tie.fit_report_device(*args)
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
tie.fit_report_device(*args)
b.record()
torch.cuda.synchronize()
print("fit_report ms", a.elapsed_time(b))
