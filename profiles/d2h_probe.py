"""Round 2: device->host copy bandwidth of 8 GiB into one pinned buffer
(the e2e leg's bound), one stream vs several copy streams, chunk sizes."""
import json
import time

import torch

N = 8 << 30
dev = torch.empty(N // 8, dtype=torch.int64, device="cuda")
dev.fill_(1)
host = torch.empty(N // 8, dtype=torch.int64, pin_memory=True)
torch.cuda.synchronize()
for nstreams in (1, 2, 4):
    for chunk_mb in (64, 256, 1024):
        ce = chunk_mb << 17  # elements
        streams = [torch.cuda.Stream() for _ in range(nstreams)]
        best = 1e9
        for rep in range(3):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            for i, a in enumerate(range(0, N // 8, ce)):
                s = streams[i % nstreams]
                with torch.cuda.stream(s):
                    host[a:a + ce].copy_(dev[a:a + ce], non_blocking=True)
            torch.cuda.synchronize()
            best = min(best, time.perf_counter() - t0)
        print(json.dumps({"streams": nstreams, "chunk_mb": chunk_mb, "GBps": round(N / best / 1e9, 2)}), flush=True)
