"""Step-by-step GPU bring-up check (prints per-stage status; run under `timeout`)."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2602_00397_b200 as ff
from oracle import ffwd_oracle as orc
from tests.fixtures import load_case

def rel(a, b):
    a = np.asarray(a, np.float64); b = np.asarray(b, np.float64)
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-30)

print(torch.cuda.get_device_name(0), flush=True)
for name in sys.argv[1:] or ["tiny_all"]:
    c = load_case(name)
    dp = ff.DevicePredictor.from_params(ff.PredictorParams(**c["pred"]), "cuda")
    x = torch.from_numpy(c["x"]).to("cuda", torch.bfloat16)
    sb = c["sparse_blocks"]
    s = ff.predictor_scores(dp, x, int(sb[0]), int(sb.size)); torch.cuda.synchronize()
    diff = (s.cpu().numpy().view(np.uint32) != c["scores"].view(np.uint32)).sum()
    print(f"[{name}] predictor: {diff} score bits differ of {s.numel()}", flush=True)
    from paper_2602_00397_b200.sparse import topk_device
    idx = topk_device(s, c["k"]).cpu().numpy()
    print(f"[{name}] topk equal: {np.array_equal(idx, c['indices'])}", flush=True)
    if c["lw"] is None:
        continue
    lw = c["lw"]
    packed = ff.pack_layer(lw["w_gate"], lw["w_up"], lw["w_down"], None, device="cuda")
    t0 = time.time()
    y = ff.dense_ffn(x, packed); torch.cuda.synchronize()
    want = orc.dense_ffn(c["x"], lw["w_gate"], lw["w_up"], lw["w_down"])
    print(f"[{name}] dense_ffn rel {rel(y.cpu().numpy(), want):.3e} ({time.time()-t0:.2f}s)", flush=True)
    comp = ff.CompensatorParams(**c["comp"])
    packed = ff.pack_layer(lw["w_gate"], lw["w_up"], lw["w_down"], comp, device="cuda")
    y, idx = ff.sparse_ffn_layer(x, packed, dp, c["k"], dense_first_last=c["dense_first_last"], return_indices=True)
    torch.cuda.synchronize()
    got = y.cpu().numpy()
    got = got[c["y_rows"]] if "y_rows" in c else got
    print(f"[{name}] layer rel {rel(got, c['y']):.3e} idx_equal {np.array_equal(idx.cpu().numpy(), c['indices'])}", flush=True)
