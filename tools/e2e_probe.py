import time, numpy as np, torch, sys
sys.path.insert(0, '/root/repo')
import paper_1810_03099_b200 as R
from paper_1810_03099_b200 import corpus as C
cp, cfg = C.config_corpus('c1')
refs = C.sample_refs(cfg['ref_seed'], cp.n_docs, cfg['K'])
ctx = R.Context(0)
tok_pin = torch.from_numpy(cp.tokens.view(np.int32)).pin_memory()
tok_np = tok_pin.numpy().view(np.uint32)
off = cp.doc_off
ctx.load_corpus(tok_np, off, cp.vocab); ctx.count(R.WEIGHT_TFIDF); ctx.set_reference_docs(refs); ctx.sign(fetch=False)
n = ctx.mrc_pairs_rows(0.99, 0, cp.n_docs, fetch=False)
out = torch.empty(int(n*1.1)+1024, dtype=torch.int64).pin_memory().numpy().view(np.uint64)
for it in range(6):
    t = [time.perf_counter()]
    ctx.load_corpus(tok_np, off, cp.vocab); ctx.synchronize(); t.append(time.perf_counter())
    ctx.count(R.WEIGHT_TFIDF); ctx.synchronize(); t.append(time.perf_counter())
    ctx.set_reference_docs(refs); ctx.synchronize(); t.append(time.perf_counter())
    ctx.sign(fetch=False); ctx.synchronize(); t.append(time.perf_counter())
    k = ctx.mrc_pairs_rows(0.99, 0, cp.n_docs, out=out); t.append(time.perf_counter())
    print(' '.join(f'{(b-a)*1e3:.3f}' for a,b in zip(t,t[1:])), f'total {(t[-1]-t[0])*1e3:.3f} ms')
# raw copy bandwidths
d = torch.empty(len(tok_np), dtype=torch.int32, device='cuda')
torch.cuda.synchronize(); a=time.perf_counter(); d.copy_(tok_pin, non_blocking=True); torch.cuda.synchronize(); b=time.perf_counter()
print('H2D GB/s', tok_pin.numel()*4/(b-a)/1e9)
o = torch.empty(len(out), dtype=torch.int64, device='cuda'); op = torch.from_numpy(out.view(np.int64))
torch.cuda.synchronize(); a=time.perf_counter(); op.copy_(o, non_blocking=True); torch.cuda.synchronize(); b=time.perf_counter()
print('D2H GB/s', o.numel()*8/(b-a)/1e9)
