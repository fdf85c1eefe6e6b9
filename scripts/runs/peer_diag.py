import sys, time, torch
sys.path.insert(0, ".")
import paper_1903_03640_b200 as tcr, tcr_inputs as gen
tcr.tcr_set_config(tcr.TCR_CFG_PEER_TIMEOUT_MS, 2000)
boxes = [tcr.tcr_peer_mailbox_alloc() for _ in range(8)]
for lg, P in ((27, 8), (30, 8), (33, 8)):
    n = 1 << lg
    x = gen.generate_tensor(gen.SEED_C4, 0, n, gen.UNIFORM_PM1)
    o32 = torch.empty(P, dtype=torch.float32, device="cuda")
    for eb in (0, 1):
        tcr.tcr_set_config(tcr.TCR_CFG_EXACT_BULK, eb)
        t0 = time.time()
        tcr.tcr_reduce_sum_exact_peer_emulated(x, boxes[:P], out_f32=o32)
        torch.cuda.synchronize()
        print(f"2^{lg} P={P} eb={eb}: {time.time()-t0:.3f} s  out={o32.cpu().tolist()[:2]}  err={[tcr.tcr_peer_mailbox_error(b) for b in boxes[:P]]}", flush=True)
    del x; torch.cuda.empty_cache()
