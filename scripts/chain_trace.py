"""Per-CTA tile timeline of the persistent forward chain (SDN_CHAIN_TRACE).
Run: SDN_NO_GRAPH=1 SDN_CHAIN_TRACE=/tmp/ct.bin python scripts/profile_step.py --steps 3
then: python scripts/chain_trace.py /tmp/ct.bin [CG]   (CG = CTAs per slot: 2 with CTA pairs, the default)"""
import sys
import numpy as np
raw = open(sys.argv[1], "rb").read()
off, recs = 0, []
while off < len(raw):
    grid, tpl, L = np.frombuffer(raw, np.int64, 3, off)
    off += 24
    n = int(grid) * 32 * 8
    st = np.frombuffer(raw, np.uint64, n, off).reshape(int(grid), 32, 8).astype(np.int64)
    off += 8 * n
    recs.append((int(grid), int(tpl), int(L), st))
grid, tpl, L, st = recs[-1]
CG = int(sys.argv[2]) if len(sys.argv) > 2 else 2
slots = grid // CG
t0 = st[st > 0].min()
us = lambda x: (x - t0) / 1e3
print(f"grid {grid}, tiles/layer {tpl}, layers {L}")
mma = []; epi = []; wait = []; gap = []
for c in range(grid):
    for i in range(32):
        g = c // CG + i * slots
        if g >= tpl * L: break
        s = st[c, i]
        if s[5] == 0: continue
        wait.append((s[1] - s[0]) / 1e3); mma.append((s[3] - s[2]) / 1e3); epi.append((s[5] - s[4]) / 1e3)
end = max(us(st[c, i, 5]) for c in range(grid) for i in range(32) if st[c, i, 5])
print(f"kernel span ~{end:.1f} us; per tile: MMA {np.mean(mma):.2f} (max {np.max(mma):.2f}), "
      f"epilogue {np.mean(epi):.2f} (max {np.max(epi):.2f}), producer flag wait {np.mean(wait):.2f} (max {np.max(wait):.2f}) us")
for c in (0, 1, 60, 107, 108, 127, 147):
    if c >= grid: continue
    line = []
    for i in range(32):
        g = c // CG + i * slots
        if g >= tpl * L: break
        s = st[c, i]
        line.append(f"L{g // tpl}t{g % tpl}: w{us(s[0]):.0f}-{us(s[1]):.0f} m{us(s[2]):.0f}-{us(s[3]):.0f} e{us(s[4]):.0f}-{us(s[5]):.0f}")
    print(f"CTA {c}: " + " | ".join(line))
