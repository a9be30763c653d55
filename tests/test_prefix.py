"""§8f-3: prefix reuse of quantized pages (chained block keys, natively
computed, pinned to the reference's hash) and the pinned-host tier for evicted
pages (payload round trips bit-identically)."""
import json
import random
import sys
from pathlib import Path

import numpy as np
import pytest
import torch

import oracle as O
from kvq_testutil import bf16_bits, make_kv
from paper_2605_29639_b200 import KVCacheSpec
from paper_2605_29639_b200.cache import BlockAllocator, block_hashes
from paper_2605_29639_b200.prefix import PrefixKVCache


def _servesim():
    try:
        import servesim  # noqa: F401
        return True
    except ImportError:
        p = Path("/root/reference/pkg/src")
        if p.exists():
            sys.path.insert(0, str(p))
            return True
    return False


def test_native_hash_matches_reference_golden():
    # frozen value of the reference (servesim test_blocks.py:63-66)
    assert block_hashes(list(range(64)), 64)[0] == 0x2802AC7B2ECBBD54
    assert block_hashes(list(range(10)), 16) == []          # partial block: no key
    keys = block_hashes(list(range(48)), 16)
    assert keys[1:] == block_hashes(list(range(16, 48)), 16, prev_key=keys[0])  # chaining


@pytest.mark.skipif(not _servesim(), reason="reference not importable")
def test_native_hash_matches_reference_implementation():
    from servesim.blocks import generate_hash_keys
    rng = random.Random(7)
    for bs in (16, 64):
        toks = [rng.randrange(0, 1 << 40) for _ in range(517)]
        assert block_hashes(toks, bs) == generate_hash_keys(toks, bs)


def fill(pkv, slots, k, v, kvo):
    pool = pkv.cache.pool.numpy()
    O.quant_append(bf16_bits(k), bf16_bits(v), np.asarray(slots, np.int32), kvo, pool)


def test_prefix_pages_are_shared_not_recomputed():
    spec = KVCacheSpec(2, kv_dtype="int8")
    pkv = PrefixKVCache(spec, 64, device="cpu")
    a = list(range(1000, 1100))
    cached, slots = pkv.admit("A", a)
    assert cached == 0 and len(slots) == 100
    k, v = make_kv(100, 2, 1), make_kv(100, 2, 2, kind="v")
    fill(pkv, slots, k, v, O.INT8)
    blocks_a = pkv.alloc.block_ids("A")
    pkv.free("A")                                   # hashed full pages stay cached
    b = a[:70] + list(range(5000, 5030))
    cached, slots_b = pkv.admit("B", b)
    assert cached == 64                             # 4 full pages of the common 70-token prefix
    assert pkv.alloc.block_ids("B")[:4] == blocks_a[:4]
    assert len(slots_b) == 100 - 64
    assert pkv.stats()["gpu_hit_tokens"] == 64
    pkv.alloc.check_invariants()
    c = list(range(1000, 1032)) + [7]               # diverges inside page 2: only pages 0-1 shared
    assert pkv.admit("C", c)[0] == 32
    pkv.alloc.check_invariants()


def test_eviction_offloads_to_host_and_promotion_restores_bytes():
    spec = KVCacheSpec(2, kv_dtype="fp8_e4m3")
    pkv = PrefixKVCache(spec, 12, device="cpu", host_blocks=16)
    a = list(range(200, 328))                       # 128 tokens = 8 pages
    _, slots = pkv.admit("A", a)
    fill(pkv, slots, make_kv(128, 2, 5), make_kv(128, 2, 6, kind="v"), O.FP8_E4M3)
    pages_a = pkv.cache.pool[torch.as_tensor(pkv.alloc.block_ids("A"))].clone()
    pkv.free("A")
    other = list(range(9000, 9000 + 160))           # 10 pages: evicts A's cached pages
    _, s2 = pkv.admit("X", other)
    fill(pkv, s2, make_kv(160, 2, 7), make_kv(160, 2, 8, kind="v"), O.FP8_E4M3)
    assert pkv.stats()["host_offloaded"] >= 6
    pkv.free("X")
    cached, rest = pkv.admit("A2", a + [1, 2, 3])
    assert cached == 128 and len(rest) == 3
    st = pkv.stats()
    assert st["host_hit_tokens"] >= 96
    got = pkv.cache.pool[torch.as_tensor(pkv.alloc.block_ids("A2")[:8])]
    assert torch.equal(got, pages_a), "promoted pages must be bit-identical"
    pkv.alloc.check_invariants()


@pytest.mark.parametrize("seed", range(4))
def test_random_prefix_workload_invariants(seed):
    rng = random.Random(seed)
    alloc = BlockAllocator(48)
    prompts = [[rng.randrange(50) for _ in range(rng.randrange(1, 90))] for _ in range(6)]
    live = {}
    for step in range(300):
        r = rng.random()
        try:
            if r < 0.45:
                sid = step
                base = rng.choice(prompts)
                toks = base[: rng.randrange(1, len(base) + 1)] + [rng.randrange(50) for _ in range(rng.randrange(0, 20))]
                cached = alloc.allocate_prefix(sid, toks)
                assert cached % 16 == 0 and cached <= len(toks)
                alloc.append_tokens(sid, toks[cached:])
                live[sid] = toks
            elif r < 0.75 and live:
                sid = rng.choice(list(live))
                extra = [rng.randrange(50) for _ in range(rng.randrange(1, 18))]
                alloc.append_tokens(sid, extra)
                live[sid] = live[sid] + extra
            elif live:
                sid = rng.choice(list(live))
                alloc.free(sid)
                del live[sid]
        except Exception as e:  # CacheThrashError under pressure is allowed; state must stay valid
            from paper_2605_29639_b200.cache import CacheThrashError
            assert isinstance(e, CacheThrashError), e
            live = {s: t for s, t in live.items() if s in alloc}
        alloc.check_invariants()
        for sid, toks in live.items():
            assert alloc.seq_len(sid) == len(toks)


GOLDEN = Path(__file__).resolve().parent / "golden"


def _pattern(k: int) -> torch.Tensor:
    from paper_2605_29639_b200._lib import PAGE_BYTES
    return ((torch.arange(PAGE_BYTES) * 7 + k * 13) % 251).to(torch.uint8).view(1, PAGE_BYTES)


@pytest.mark.parametrize("trace", range(4))
def test_host_tier_replays_reference_trace(trace):
    """The reference's own GPU + LOCAL_CPU tiers with writeback_on_evict
    (tests/golden/ref_host_trace.json, made by servesim.tiered_cache): demotion
    only when absent and only without cascading (tiered_cache.py:254-275),
    promotion keeps the host copy (277-317).  Replayed through PrefixKVCache's
    own eviction hook and _promote, with every page's bytes checked after each
    promotion (a promoted page must carry its own key's bytes)."""
    from paper_2605_29639_b200.cache import CacheThrashError
    tr = json.loads((GOLDEN / "ref_host_trace.json").read_text())[trace]
    pkv = PrefixKVCache(KVCacheSpec(1), tr["gpu_blocks"], device="cpu", host_blocks=tr["cpu_blocks"])
    pool = pkv.alloc.pool
    for i, rec in enumerate(tr["ops"]):
        k, clock = rec["key"], rec["clock"]
        key = ("h", k)
        pkv.alloc.clock = clock
        hit = None
        try:
            if rec["op"] == "insert":
                pkv.cache.pool[pool.insert(key, 16, clock)] = _pattern(k)
            elif rec["op"] == "fetch":
                if pool.entry(key) is not None:
                    hit = "GPU"
                elif key in pkv.host:
                    hit = "LOCAL_CPU"
                    assert pkv._promote(key)
                    assert torch.equal(pkv.cache.pool[pool.lookup(key)], _pattern(k)), (i, "promoted bytes")
                if hit is not None:
                    pool.acquire(key, clock)
            elif rec["op"] == "release":
                pool.release([key], clock)
            elif rec["op"] == "evict":
                assert pool.evict(1) == [("h", e) for e in rec["evicted"]], i
            outcome = "ok"
        except CacheThrashError as e:
            outcome = f"thrash:{e.bytes_needed // pool.bytes_per_block}"
        except ValueError as e:
            outcome = f"ValueError:{e}"
        except KeyError:
            outcome = "KeyError"
        assert outcome == rec["outcome"], (i, rec, outcome)
        if "hit" in rec:
            assert hit == rec["hit"], (i, rec, hit)
        assert {str(kk[1]): e.ref_count for kk, e in pool._entries.items()} == rec["gpu"], (i, rec)
        assert sorted(kk[1] for kk in pkv.host.keys()) == rec["cpu"], (i, rec)


def test_decoding_without_token_ids_stops_prefix_hashing():
    """A prefix-admitted sequence decoded with append_one (ids unknown) must not
    key the pages it fills: a later prompt sharing only the admitted tokens
    reuses the admitted full pages and nothing past them."""
    spec = KVCacheSpec(1)
    pkv = PrefixKVCache(spec, 32, device="cpu")
    a = list(range(100, 140))                       # 2 full pages + 8 tokens
    assert pkv.admit("A", a)[0] == 0
    for _ in range(8):                              # fills page 2 with decoded tokens
        pkv.alloc.append_one(["A"])
    pkv.alloc.append_slots("A", 20)                 # and pages past it
    pkv.free("A")
    b = a + [7] * 8                                 # same 40 tokens, different 8 after them
    cached, _ = pkv.admit("B", b)
    assert cached == 32
    pkv.alloc.check_invariants()
    with pytest.raises(ValueError, match="without token ids"):
        pkv.alloc.allocate("C")
        pkv.alloc.append_slots("C", 3)
        pkv.alloc.append_tokens("C", [1, 2])


def test_admit_releases_everything_on_thrash():
    """CacheThrashError inside admit leaves no sequence and no extra references
    (the reference releases what it acquired, simulator.py:397-400), so the
    request can be retried."""
    from paper_2605_29639_b200.cache import CacheThrashError
    pkv = PrefixKVCache(KVCacheSpec(1), 6, device="cpu")
    shared = list(range(500, 532))                  # 2 pages, cached after free
    pkv.admit("P", shared)
    pkv.alloc.allocate("hog")
    pkv.alloc.append_slots("hog", 3 * 16)           # 3 private pages pinned
    pkv.free("P")
    refs = [pkv.alloc.ref_count(b) for b in range(6)]
    with pytest.raises(CacheThrashError):
        pkv.admit("R", shared + list(range(64)))    # shares 2 pages, then needs 4 more of 1 free
    assert "R" not in pkv.alloc
    assert [pkv.alloc.ref_count(b) for b in range(6)] == refs
    pkv.alloc.check_invariants()
    pkv.free("hog")
    assert pkv.admit("R", shared + list(range(64)))[0] == 32   # the retry succeeds


def test_promotion_with_a_one_block_host_tier():
    """The promoted page keeps its own bytes when the GPU insert behind the
    promotion evicts (and tries to demote) another page into a full host tier."""
    pkv = PrefixKVCache(KVCacheSpec(1), 1, device="cpu", host_blocks=1)
    pool = pkv.alloc.pool
    pkv.cache.pool[pool.insert(("h", 1), 16, 1)] = _pattern(1)
    pool.evict(1)                                    # ("h", 1) demoted into the single host slot
    pkv.cache.pool[pool.insert(("h", 2), 16, 2)] = _pattern(2)
    assert pkv._promote(("h", 1))                    # evicts ("h", 2): host full, dropped
    assert torch.equal(pkv.cache.pool[pool.lookup(("h", 1))], _pattern(1))
    assert pkv.host.keys() == [("h", 1)] and pkv.host.dropped == 1
