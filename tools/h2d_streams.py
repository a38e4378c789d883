"""Diagnostics: pinned host -> HBM bandwidth with 1, 2, 4, 8 concurrent copy
streams (chunked), CUDA events around the whole transfer.
    python tools/h2d_streams.py"""
import json


def main():
    import torch
    n = 4 << 30
    h = torch.empty(n, dtype=torch.uint8, pin_memory=True)
    d = torch.empty(n, dtype=torch.uint8, device="cuda:0")
    out = {}
    for k in (1, 2, 4, 8):
        streams = [torch.cuda.Stream() for _ in range(k)]
        best = 1e9
        for _ in range(3):
            torch.cuda.synchronize()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            chunk = n // k
            for i, s in enumerate(streams):
                s.wait_event(a)
                with torch.cuda.stream(s):
                    d[i * chunk:(i + 1) * chunk].copy_(h[i * chunk:(i + 1) * chunk], non_blocking=True)
            for s in streams:
                torch.cuda.current_stream().wait_stream(s)
            b.record()
            torch.cuda.synchronize()
            best = min(best, a.elapsed_time(b))
        out[f"streams{k}"] = n / (best / 1e3) / 1e9
    print(json.dumps(out))


if __name__ == "__main__":
    main()
