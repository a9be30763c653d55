import sys, torch, numpy as np
sys.path.insert(0, '.')
import bench
from paper_2605_29639_b200 import KVCacheSpec, PagedKVCache, ops
dev = torch.device('cuda:0')
cfg = bench.CONFIGS['c2']
lens = bench.ctx_lens(cfg) + 1
nblk = -(-lens // 16); NB = int(nblk.sum()); mb = int(nblk.max())
B, Hq, Hkv = 256, 32, 8
pool = torch.randint(0, 256, (NB, Hkv, 4224), dtype=torch.uint8, device=dev)
pool[..., 4096:] = torch.full((NB, Hkv, 32), 0.02, device=dev).view(torch.uint8).view(NB, Hkv, 128)
cache = PagedKVCache(KVCacheSpec(Hkv), NB, device=dev, pool=pool)
perm = np.random.default_rng(7).permutation(NB).astype(np.int32)
table = np.zeros((B, mb), np.int32); pos = 0
for b in range(B):
    table[b, :nblk[b]] = perm[pos:pos + nblk[b]]; pos += nblk[b]
table_d = torch.from_numpy(table).to(dev); lens_d = torch.from_numpy(lens.astype(np.int32)).to(dev)
slots = torch.from_numpy((table[np.arange(B), (lens - 1) // 16].astype(np.int64) * 16 + (lens - 1) % 16).astype(np.int32)).to(dev)
q = torch.randn((B, Hq, 128), device=dev).to(torch.bfloat16)
k = torch.randn((B, Hkv, 128), device=dev).to(torch.bfloat16); v = torch.randn_like(k)
out = torch.empty((Hq, B, 128), dtype=torch.bfloat16, device=dev)
pps = ops.pages_per_split(B, Hkv, NB, mb)
ws = torch.zeros(ops.workspace_bytes(B, Hq, Hkv, -(-mb // pps)), dtype=torch.uint8, device=dev)
step = lambda: ops.decode_step(cache, k, v, slots, q, table_d, lens_d, out=out, head_major=True, pages_per_split=pps, workspace=ws, append_tail_only=True)
step(); torch.cuda.synchronize()
g1 = torch.cuda.CUDAGraph()
with torch.cuda.graph(g1): step()
gN = torch.cuda.CUDAGraph()
with torch.cuda.graph(gN):
    for _ in range(50): step()
def t(fn, n):
    fn(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); [fn() for _ in range(n)]; e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n * 1e3
print(f"unrolled graph: {t(gN.replay, 4) / 50:.1f} us/step; one graph per step: {t(g1.replay, 200):.1f} us/step")
