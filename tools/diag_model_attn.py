"""Diagnose the sparse attention cost inside the NEXT-4 model: time the fused
decode layer on the model's own queries vs random queries, right after the
prompt and after n generated tokens, and count fused launches."""
import ctypes, os, sys
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2602_03184_b200 import dynsplit as D
from paper_2602_03184_b200.model import LlamaShape, RandomLlama
from synth import generators as G
dev = torch.device("cuda:0")
B = int(sys.argv[1]) if len(sys.argv) > 1 else 1
NL, S0, S_cap, budget = 4, 32768, 32768 + 2100, 2048
ids = torch.from_numpy(G.T7_IDS).to(dev)
w10 = torch.from_numpy(np.tile(G.T7_W10, (B, 1))).to(torch.uint8)
cfg = D.default_config(page_cap=(S_cap // 16) + D.max_blocks(S_cap, D.default_config()) // 2 + 64)
m = RandomLlama(LlamaShape(layers=NL), B, S_cap, budget, dev, seed=1, cfg=cfg, delim_ids=ids, w10=w10)
toks = torch.from_numpy(np.stack([G.tokens(9000 + b, S0) for b in range(B)])).to(dev)
m.prefill_synthetic(toks, seed=2)
lib = D.lib()
lib.dynsplit_debug_fused_launches.restype = ctypes.c_longlong
saved = []
orig = D.decode_layer
def spy(q, lay, budget, out=None, ws=None):
    saved.append(q.clone())
    return orig(q, lay, budget, out=out, ws=ws)
D.decode_layer = spy


def time_layers(qs, dense=False, reps=20):
    def run():
        for l in range(NL):
            if dense:
                D.decode_attn(qs[l], m.layers[l], None, out=(m.o, m.lse), ws=m.ws_dec)
            else:
                orig(qs[l], m.layers[l], budget, out=(m.ns, m.mg, m.kp, m.wl, m.o, m.lse), ws=m.ws_dec)
    run(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        run()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps / NL * 1e3


tok = toks[:, -1].contiguous()
for phase, n in (("prompt", 1), ("+1000", 1000), ("+2000", 1000)):
    for _ in range(n):
        saved.clear()
        tok = m.step(tok)
    torch.cuda.synchronize()
    qs = [s.clone() for s in saved]
    c0 = lib.dynsplit_debug_fused_launches()
    t_model = time_layers(qs)
    c1 = lib.dynsplit_debug_fused_launches()
    g = torch.Generator(device=dev); g.manual_seed(5)
    qr = [torch.randn(B, 32, 128, generator=g, device=dev).to(torch.bfloat16) for _ in range(NL)]
    t_rand = time_layers(qr)
    t_dense = time_layers(qs, dense=True)
    qn = [float(q.float().norm(dim=-1).mean()) for q in qs]
    nsel = m.ns.float().mean().item()
    print(f"{phase}: pos {int(m.pos.item())} nb {m.layers[0].n_blocks.tolist()[:2]}  fused launches/layer-call "
          f"{(c1 - c0) / (21 * NL):.2f}  us/layer: model-q {t_model:.1f}  random-q {t_rand:.1f}  dense {t_dense:.1f}"
          f"  |q| {qn[0]:.1f}  mean n_sel {nsel:.0f}  err {D.read_device_error(m.ws_dec)}", flush=True)
    if os.environ.get("DYNSPLIT_DEBUG_BUILD"):
        NAMES = ["start", "plan", "pdl_wait", "scored+arrive A", "A passed", "range classified", "B passed+gathered",
                 "band selected", "bits final", "union counted", "dealt", "pages done", "merged", "B passed",
                 "q loaded", "digests in smem"]
        dbg = torch.zeros(148 * 64, dtype=torch.int64, device=dev)
        lib.dynsplit_debug_fused_timer.argtypes = [ctypes.c_void_p]
        lib.dynsplit_debug_fused_timer(ctypes.c_void_p(dbg.data_ptr()))
        orig(qs[0], m.layers[0], budget, out=(m.ns, m.mg, m.kp, m.wl, m.o, m.lse), ws=m.ws_dec)
        torch.cuda.synchronize()
        lib.dynsplit_debug_fused_timer(ctypes.c_void_p(0))
        tc = dbg.view(148, 64).cpu().numpy().astype(np.float64)
        used = tc[:, 0] > 0
        t = tc[used, :16]
        t0 = t[:, 0].min()
        for k in [0, 1, 2, 14, 15, 3, 4, 5, 13, 7, 8, 9, 10, 11, 12]:
            col = t[:, k]
            col = col[col > 0]
            if len(col):
                r = (col - t0) / 1e3
                print(f"   {k:2d} {NAMES[k]:18s} n={len(col):3d} min {r.min():7.2f} p50 {np.median(r):7.2f} max {r.max():7.2f}")
        ex = dbg.view(148, 64)[:, 32:52].cpu().numpy()[used]
        fbk = ex[:, 16:20]
        sx = dbg.view(148, 64)[:, 56:60].cpu().numpy().astype(np.float64)[used]
        if (sx[:, 0] > 0).any():
            ok = sx[:, 0] > 0
            print("   fallback stamps (us after 'band selected' p50):",
                  [f"{np.median((sx[ok, k] - tc[used][ok, 7]) / 1e3):.2f}" for k in range(4)])
        print(f"   fallback CTAs per head {[(int((fbk[:, g] > 0).sum())) for g in range(4)]}  band in bin j* max "
              f"{[int(fbk[:, g].max()) - 1 for g in range(4)]}")
        for g2 in range(4):
            nb_, ov, wh, wb = ex[:, 4 * g2], ex[:, 4 * g2 + 1], ex[:, 4 * g2 + 2], ex[:, 4 * g2 + 3]
            print(f"   head {g2}: nband min {nb_.min()} max {nb_.max()}  over {int(ov.sum())}  W_hi {wh.min()}-{wh.max()}"
                  f"  W_bd {wb.min()}-{wb.max()}")
        print("   n_sel per head", m.ns[0].tolist()[:8], "marg", m.mg[0].tolist()[:4], "keep", m.kp[0].tolist()[:4], flush=True)
