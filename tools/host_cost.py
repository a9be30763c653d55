"""Host cost of an eager op call (a 1-page decode: the GPU work is negligible, so
the loop is host-bound), plus a cProfile breakdown of the Python wrapper."""
import sys, time, torch
sys.path.insert(0, '.')
from paper_2605_29639_b200 import KVCacheSpec, PagedKVCache, paged_decode_attention
dev = torch.device('cuda:0')
cache = PagedKVCache(KVCacheSpec(8), 64, device=dev)
cache.pool[..., 4096:] = 0
q = torch.randn((1, 32, 128), device=dev).to(torch.bfloat16)
table = torch.zeros((1, 4), dtype=torch.int32, device=dev); lens = torch.tensor([15], dtype=torch.int32, device=dev)
out = torch.empty((1, 32, 128), dtype=torch.bfloat16, device=dev)
for _ in range(50): paged_decode_attention(q, cache, table, lens, out=out, pages_per_split=8)
torch.cuda.synchronize()
n = 2000
t = time.perf_counter()
for _ in range(n): paged_decode_attention(q, cache, table, lens, out=out, pages_per_split=8)
torch.cuda.synchronize()
print(f"eager paged_decode_attention (1 page): {(time.perf_counter() - t) / n * 1e6:.1f} us per call (host-bound)")

import cProfile, pstats
cProfile.run("for _ in range(2000): paged_decode_attention(q, cache, table, lens, out=out, pages_per_split=8)", "/tmp/hc.prof")
pstats.Stats("/tmp/hc.prof").sort_stats("tottime").print_stats(12)
