"""PCIe copy-engine probe (dev tool, one B200): H2D and D2H throughput from / to pinned host
memory, alone and concurrent, with 1 / 2 / 4 streams per direction — does splitting the
host-fed step's copies over more copy engines move more bytes per second?"""
import json

import torch

GB = 1 << 30


def run(n_streams, nbytes, h2d=True, d2h=True, reps=3):
    dev = torch.device("cuda")
    hs = [torch.empty(nbytes // n_streams, dtype=torch.uint8).pin_memory() for _ in range(n_streams)]
    ho = [torch.empty(nbytes // n_streams, dtype=torch.uint8).pin_memory() for _ in range(n_streams)]
    ds = [torch.empty(nbytes // n_streams, dtype=torch.uint8, device=dev) for _ in range(n_streams)]
    do = [torch.ones(nbytes // n_streams, dtype=torch.uint8, device=dev) for _ in range(n_streams)]
    st_in = [torch.cuda.Stream() for _ in range(n_streams)]
    st_out = [torch.cuda.Stream() for _ in range(n_streams)]
    best = None
    for _ in range(reps):
        torch.cuda.synchronize()
        s, e = torch.cuda.Event(True), torch.cuda.Event(True)
        s.record()
        cur = torch.cuda.current_stream()
        for i in range(n_streams):
            if h2d:
                st_in[i].wait_stream(cur)
                with torch.cuda.stream(st_in[i]):
                    ds[i].copy_(hs[i], non_blocking=True)
            if d2h:
                st_out[i].wait_stream(cur)
                with torch.cuda.stream(st_out[i]):
                    ho[i].copy_(do[i], non_blocking=True)
        for i in range(n_streams):
            if h2d:
                cur.wait_stream(st_in[i])
            if d2h:
                cur.wait_stream(st_out[i])
        e.record()
        torch.cuda.synchronize()
        ms = s.elapsed_time(e)
        best = ms if best is None else min(best, ms)
    return best


def main():
    nbytes = 4 * GB
    for n in (1, 2, 4):
        for mode in ("h2d", "d2h", "both"):
            ms = run(n, nbytes, h2d=mode in ("h2d", "both"), d2h=mode in ("d2h", "both"))
            print(json.dumps({"streams_per_direction": n, "mode": mode, "ms": round(ms, 2),
                              "GB_s_per_direction": round(nbytes / ms / 1e6, 1)}), flush=True)


if __name__ == "__main__":
    main()
