"""Block lifecycle and allocator: the reference's GPU-tier rules replayed from
traces the reference itself produced (tests/golden/ref_block_trace.json, made by
servesim.tiered_cache.TieredCacheStore), the reference's own fixtures
(test_tiered_cache.py:130-142, 220-233) restated, and randomized op sequences
against a shadow model (after test_tiered_cache.py:243-327)."""
import json
import random
from pathlib import Path

import pytest

from paper_2605_29639_b200.cache import BlockAllocator, BlockPool, CacheThrashError

GOLDEN = Path(__file__).resolve().parent / "golden"
SIZE = 4224


@pytest.mark.parametrize("trace", range(4))
def test_replay_reference_trace(trace):
    tr = json.loads((GOLDEN / "ref_block_trace.json").read_text())[trace]
    pool = BlockPool(tr["cap_blocks"], 16, bytes_per_block=SIZE)
    for i, rec in enumerate(tr["ops"]):
        op, k, clock = rec["op"], rec["key"], rec["clock"]
        try:
            if op == "insert":
                pool.insert(k, rec["watermark"], clock)
            elif op == "acquire":
                pool.acquire(k, clock)
            elif op == "release":
                pool.release([k], clock)
            elif op == "watermark":
                pool.set_watermark(k, rec["watermark"])
            elif op == "evict":
                got = pool.evict(rec["nblocks"])
                assert got == rec["evicted"], (i, got, rec["evicted"])
            outcome = "ok"
        except CacheThrashError as e:
            outcome = f"thrash:{e.bytes_needed // SIZE}"
        except ValueError as e:
            outcome = f"ValueError:{e}"
        except KeyError:
            outcome = "KeyError"
        assert outcome == rec["outcome"], (i, rec, outcome)
        state = {str(key): [e.ref_count, e.watermark] for key, e in pool._entries.items()}
        assert state == rec["state"], (i, rec)


def test_reference_fixture_rules():
    # test_tiered_cache.py:130-135 partial block is exclusive
    p = BlockPool(10)
    p.insert(0xA, 8)
    p.acquire(0xA)
    with pytest.raises(ValueError, match="exclusive"):
        p.acquire(0xA)
    # :137-142 full block allows concurrent refs
    p.insert(0xB, 16)
    p.acquire(0xB)
    p.acquire(0xB)
    assert p.entry(0xB).ref_count == 2
    # :220-233 watermark only grows, then the full block becomes shareable
    p.set_watermark(0xA, 12)
    with pytest.raises(ValueError):
        p.set_watermark(0xA, 10)
    with pytest.raises(ValueError):
        p.set_watermark(0xA, 17)
    p.set_watermark(0xA, 16)
    p.release([0xA])
    p.acquire(0xA)
    p.acquire(0xA)
    with pytest.raises(ValueError, match="double release"):
        p.release([0xC])


def test_append_fork_free_basics():
    a = BlockAllocator(8)
    a.allocate("p")
    slots = a.append_slots("p", 20)
    assert slots == list(range(16)) + [16, 17, 18, 19]
    copies = a.fork("p", "c")          # full block shared, partial tail copied
    assert copies == [(1, 2)]
    assert a.block_ids("c") == [0, 2] and a.ref_count(0) == 2 and a.ref_count(1) == 1
    assert a.append_slots("c", 13) == [36, 37, 38, 39, 40, 41, 42, 43, 44, 45, 46, 47, 48]
    assert a.block_ids("c") == [0, 2, 3]
    a.check_invariants()
    a.free("p")
    assert a.ref_count(0) == 1 and a.ref_count(1) == 0
    a.free("c")
    assert a.num_free == 8
    a.check_invariants()


def test_fork_of_block_aligned_parent_copies_nothing():
    a = BlockAllocator(8)
    a.allocate(0)
    a.append_slots(0, 32)
    assert a.fork(0, 1) == []
    assert a.append_slots(1, 1) == [32]          # new private block, shared ones untouched
    assert a.block_ids(0) == [0, 1] and a.block_ids(1) == [0, 1, 2]
    a.check_invariants()


def test_thrash_is_atomic():
    a = BlockAllocator(3, bytes_per_block=SIZE)
    a.allocate(0)
    a.append_slots(0, 40)
    with pytest.raises(CacheThrashError) as ei:
        a.append_slots(0, 20)          # needs 2 new blocks, 0 free
    assert ei.value.bytes_needed == SIZE
    assert a.seq_len(0) == 40
    a.check_invariants()


@pytest.mark.parametrize("seed", range(6))
def test_random_ops_shadow_model(seed):
    rng = random.Random(seed)
    a = BlockAllocator(64)
    shadow = {}          # seq -> list of logical token ids (to check slot stability)
    slot_of = {}         # (seq, pos) -> slot
    next_id = 0
    for _ in range(1500):
        op = rng.random()
        live = list(shadow)
        try:
            if op < 0.2 or not live:
                a.allocate(next_id)
                shadow[next_id] = 0
                next_id += 1
            elif op < 0.65:
                s = rng.choice(live)
                n = rng.choice([1, 1, 1, 3, 16, 17, 40])
                slots = a.append_slots(s, n)
                assert len(slots) == n and len(set(slots)) == n
                for i, sl in enumerate(slots):
                    slot_of[(s, shadow[s] + i)] = sl
                shadow[s] += n
            elif op < 0.8:
                s = rng.choice(live)
                copies = a.fork(s, next_id)
                L = shadow[s]
                shadow[next_id] = L
                for pos in range(L):
                    blk = slot_of[(s, pos)] // 16
                    if copies and blk == copies[0][0]:
                        slot_of[(next_id, pos)] = copies[0][1] * 16 + pos % 16
                    else:
                        slot_of[(next_id, pos)] = slot_of[(s, pos)]
                next_id += 1
            else:
                s = rng.choice(live)
                a.free(s)
                del shadow[s]
        except CacheThrashError:
            pass
        a.check_invariants()
        # every live sequence still resolves its tokens to the same slots
        for s, L in shadow.items():
            ids = a.block_ids(s)
            for pos in range(0, L, 7):
                assert ids[pos // 16] * 16 + pos % 16 == slot_of[(s, pos)]


@pytest.mark.parametrize("seed", [0, 1, 2])
def test_decode_step_fast_paths(seed):
    """append_one (the decode step's batched slots) == append_slots(s, 1) per
    sequence, and the incremental BlockTable stays equal to a full rebuild
    under joins, leaves, forks and prefills between steps."""
    import numpy as np
    from paper_2605_29639_b200.cache import BlockTable
    rng = random.Random(seed)
    a, b = BlockAllocator(600), BlockAllocator(600)      # a: fast paths, b: reference calls
    table = BlockTable(24, 64, device="cpu")
    live, nxt = [], 0
    for step in range(120):
        op = rng.random()
        if op < 0.2 or len(live) < 4:                   # join with a prefill
            n = rng.randint(0, 70)
            for x in (a, b):
                x.allocate(nxt)
                x.append_slots(nxt, n)
            live.append(nxt)
            nxt += 1
        elif op < 0.3:                                  # leave
            s = live.pop(rng.randrange(len(live)))
            a.free(s)
            b.free(s)
        elif op < 0.4:                                  # fork
            p = rng.choice(live)
            ca, cb = a.fork(p, nxt), b.fork(p, nxt)
            assert ca == cb
            live.append(nxt)
            nxt += 1
        live = live[:24]
        for s in list(a.seq_ids()):
            if s not in live:
                a.free(s)
                b.free(s)
        rng.shuffle(live)                               # rows move between sequences
        got = a.append_one(live)
        want = [b.append_slots(s, 1)[0] for s in live]
        assert got.tolist() == want
        table.sync(a, live)
        mb = 64
        full = a.block_table(live, mb)
        lens = a.seq_lens(live)
        dev = table.table.numpy()[: len(live)]
        for i, s in enumerate(live):
            n = -(-int(lens[i]) // 16)
            assert np.array_equal(dev[i, :n], full[i, :n]), (step, s)
        assert np.array_equal(table.seq_lens.numpy()[: len(live)], lens)
        a.check_invariants()
        assert a.block_table(live, mb).tolist() == b.block_table(live, mb).tolist()


def test_append_one_is_atomic_on_thrash():
    a = BlockAllocator(4)
    for s in range(4):
        a.allocate(s)
        a.append_slots(s, 16)                           # every block full: next token needs a new block
    before = [a.seq_len(s) for s in range(4)]
    with pytest.raises(CacheThrashError):
        a.append_one([0, 1, 2, 3])
    assert [a.seq_len(s) for s in range(4)] == before
    a.check_invariants()
