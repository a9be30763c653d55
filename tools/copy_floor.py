"""Floor for a K1-sized transfer on this box: torch copies of the C5 append's
bytes (34.6 MB of bf16 rows read, 17.8 MB of pages written), back to back and
with L2 flushed before each launch, CUDA events."""
import torch


def timeit(fn, flush=None, n=50):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(n):
        if flush is not None:
            flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); fn(); b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b) * 1e3)
    ts.sort()
    return ts[len(ts) // 2]


def main():
    dev = torch.device("cuda:0")
    rd = torch.empty(8444 * 8 * 512 * 2, dtype=torch.uint8, device=dev)   # K and V rows
    wr = torch.empty(8444 * 8 * 264, dtype=torch.uint8, device=dev)       # pages
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    half = rd[: wr.numel()]
    tiny = torch.empty(16, dtype=torch.uint8, device=dev)
    print(f"empty-ish launch (16-byte memset) between events: {timeit(lambda: tiny.zero_()):.2f} us")
    for name, fn, byt in (("copy 17.8 MB -> 17.8 MB", lambda: wr.copy_(half), 2 * wr.numel()),
                          ("copy 34.6 MB -> 34.6 MB", lambda: rd.view(2, -1)[1].copy_(rd.view(2, -1)[0]), rd.numel())):
        t_hot, t_cold = timeit(fn), timeit(fn, flush)
        print(f"{name}: {t_hot:.2f} us back to back ({byt / t_hot / 1e3:.0f} GB/s), "
              f"{t_cold:.2f} us cold L2 ({byt / t_cold / 1e3:.0f} GB/s)")


if __name__ == "__main__":
    main()
