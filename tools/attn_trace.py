"""Per-CTA timeline of the fused attention backward (debug hook dpn_attn_debug_trace).
Prints median cycle deltas between the stamps the kernel records (see ATTN_STAMP slots)."""
import sys, ctypes, torch
sys.path.insert(0, ".")
from paper_2505_05856_b200 import _lib, kernels as k
_lib.init_device(0)
lib = _lib.load_library()
b, h, s = 8, 16, 512
H = h * 64
qkv = (torch.randn(b * s, 3 * H, device="cuda") * 0.5).bfloat16()
out = torch.empty(b * s, H, device="cuda", dtype=torch.bfloat16)
lse = torch.empty(b, h, s, device="cuda")
dout = torch.randn(b * s, H, device="cuda").bfloat16()
dqkv = torch.empty_like(qkv)
k.attn_fwd(qkv, out, lse, b, s, h, False)
for _ in range(3):
    k.attn_bwd(qkv, out, dout, lse, dqkv, b, s, h, False)
n_cta = (s // 128) * h * b
tr = torch.zeros(n_cta, 64, dtype=torch.int64, device="cuda")
lib.dpn_attn_debug_trace.argtypes = [ctypes.c_void_p]
lib.dpn_attn_debug_trace(tr.data_ptr())
k.attn_bwd(qkv, out, dout, lse, dqkv, b, s, h, False)
torch.cuda.synchronize()
lib.dpn_attn_debug_trace(None)
t = tr.cpu()


def med(a, b_):
    v = sorted(int(x) for x in (t[:, b_] - t[:, a]))
    return v[len(v) // 2]


print("MMA: kv_full wait", med(0, 1))
for it in range(4):
    o = 2 + it * 8
    print(f"it{it}: wait sp_full {med(o, o+1)} tmem ld {med(o+1, o+2)} wait ds_empty {med(o+2, o+3)} "
          f"compute {med(o+3, o+4)} wait p_empty {med(o+4, o+5)} store P {med(o+5, o+6)}",
          f"| mma ds_full->{med(1 if it == 0 else 45+(it-1)*4, 44+it*4)} dq_empty wait {med(44+it*4, 45+it*4)}")
print("softmax loop end -> dkv", med(36, 37))
print("total CTA (mma start -> dkv done)", med(0, 37))
for it in range(3):
    print(f"it{it}->it{it+1} period", med(3 + it * 8, 3 + (it + 1) * 8))
# whole-kernel view: per-SM CTA timeline from %globaltimer
g0, g1, sm = t[:, 60], t[:, 61], t[:, 62]
print("kernel span (globaltimer) us", (int(g1.max()) - int(g0.min())) / 1e3)
durs = sorted(int(x) for x in (g1 - g0))
print("CTA duration ns: median", durs[len(durs) // 2], "min", durs[0], "max", durs[-1])
clk = [(int(t[i, 59]) - int(t[i, 63])) / max(1, int(g1[i]) - int(g0[i])) for i in range(t.shape[0])]
clk.sort()
print("SM clock GHz (median over CTAs)", round(clk[len(clk) // 2], 3))
per_sm = {}
for i in range(t.shape[0]):
    per_sm.setdefault(int(sm[i]), []).append((int(g0[i]), int(g1[i])))
gaps, counts = [], []
for k_, v in per_sm.items():
    v.sort()
    counts.append(len(v))
    for a_, b_ in zip(v, v[1:]):
        gaps.append(b_[0] - a_[1])
gaps.sort()
print("CTAs per SM: min", min(counts), "max", max(counts), "SMs used", len(per_sm))
if gaps:
    print("gap between CTAs on an SM ns: median", gaps[len(gaps) // 2], "max", gaps[-1])
