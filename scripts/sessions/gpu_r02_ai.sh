#!/bin/bash
# Round-2 GPU session AI: cost of pinned host allocation on the box (sizes the host-staged configurations use).
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
python - > gpurun_out/r02ai_pinned.log 2>&1 <<'PY'
import time, torch
torch.cuda.init()
for gb in (1, 4, 16):
    t = time.time(); x = torch.empty(gb * 2**30, dtype=torch.uint8, pin_memory=True); a = time.time() - t
    d = torch.empty(gb * 2**30, dtype=torch.uint8, device="cuda")
    torch.cuda.synchronize(); t = time.time(); d.copy_(x, non_blocking=True); torch.cuda.synchronize(); c = time.time() - t
    t = time.time(); del x; f = time.time() - t
    print(f"{gb} GB: cudaHostAlloc {a:.3f} s ({gb/a:.1f} GB/s), H2D copy {c:.3f} s ({gb/c:.1f} GB/s), free {f:.3f} s")
    del d
PY
