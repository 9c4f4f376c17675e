"""Wider randomised parity sweep than k2r_sweep.py: ARBITRARY sides (odd,
prime, not multiples of 16 -- the byte-staged and generic round paths), any
subframe count dividing the side, 1-7 rounds, PLCM and LASM keys, through
every frame entry point (per-frame host calls, batched host calls, the _wh
pad/crop calls, the device-resident call, sharded handles on repeated device
lists), each checked byte for byte against the oracle and decrypted back by a
fresh handle.  Tool, not product: the oracle is the checker here.

  python tools/wide_sweep.py [seed] [cases] [maxside] [big_every]
"""
import os, sys, random, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np
import torch
import paper_2302_07411_b200 as cve
from workloads import synth
from _oracle import Oracle

seed = int(sys.argv[1]) if len(sys.argv) > 1 else 11
cases = int(sys.argv[2]) if len(sys.argv) > 2 else 80
maxside = int(sys.argv[3]) if len(sys.argv) > 3 else 700
big_every = int(sys.argv[4]) if len(sys.argv) > 4 else 10
rng = random.Random(seed)
bad = 0
t_start = time.time()


def divisors(side, cap=256):
    return [d for d in range(1, min(side, cap) + 1) if side % d == 0]


def pick_side(it):
    kind = rng.random()
    if it % big_every == big_every - 1:  # a large one now and then
        return rng.choice([1024, 1080, 1536, 1920, 2048, 2160, 1000, 1234, 1917])
    if kind < 0.35:
        return rng.randint(1, maxside)          # anything, odd sides included
    if kind < 0.6:
        return 16 * rng.randint(1, maxside // 16)
    if kind < 0.8:
        return 3 * rng.randint(1, maxside // 3)
    return rng.choice([1, 2, 3, 5, 7, 15, 17, 31, 33, 63, 65, 127, 129, 255, 257, 479, 481, 511, 513])


def oracle_frames(key, n, r, frames):
    want = frames.copy()
    o = Oracle(key, n, r)
    for t in range(len(want)):
        assert o.encrypt(want[t]) == 0
    o.close()
    return want


for it in range(cases):
    side = pick_side(it)
    n = rng.choice(divisors(side))
    r = rng.choice([1, 2, 3, 5, 5, 5, 7])
    lasm = rng.random() < 0.25
    key = synth.det_key_lasm(seed * 1000 + it) if lasm else synth.det_key(seed * 1000 + it)
    nf = 3 if side <= 800 else 2
    frames = np.random.default_rng(seed * 77 + it).integers(0, 256, size=(nf, side, side, 3),
                                                            dtype=np.uint8)
    if rng.random() < 0.15:
        frames[0] = 0
    if rng.random() < 0.15:
        frames[-1] = 255
    want = oracle_frames(key, n, r, frames)
    mode = rng.choice(["frame", "frames", "device", "shard2", "shard3", "shard_dev", "mixed"])
    got = frames.copy()
    try:
        if mode == "frame":
            h = cve.Cipher(key, n, r)
            for t in range(nf):
                h.encrypt_frame(got[t])
        elif mode == "frames":
            cve.Cipher(key, n, r).encrypt_frames(got)
        elif mode == "device":
            d = torch.from_numpy(got).cuda()
            h = cve.Cipher(key, n, r)
            h.encrypt_frames_device(d.data_ptr(), side, nf, torch.cuda.current_stream().cuda_stream)
            torch.cuda.synchronize()
            got = d.cpu().numpy()
        elif mode in ("shard2", "shard3"):
            h = cve.Cipher(key, n, r, devices=[0] * (2 if mode == "shard2" else 3))
            for t in range(nf):
                h.encrypt_frame(got[t])
        elif mode == "shard_dev":
            G = 2
            h = cve.Cipher(key, n, r, devices=[0] * G)
            parts = [torch.from_numpy(np.ascontiguousarray(got[i::G])).cuda() for i in range(G)]
            h.encrypt_frames_sharded([p.data_ptr() for p in parts], side, nf)
            h.synchronize()
            torch.cuda.synchronize()
            for i in range(G):
                got[i::G] = parts[i].cpu().numpy()
        else:  # mixed: first frame alone, the rest batched, same handle
            h = cve.Cipher(key, n, r)
            h.encrypt_frame(got[0])
            h.encrypt_frames(got[1:])
        ok = np.array_equal(got, want)
        back = got.copy()
        dmode = rng.choice(["frames", "frame", "shard2"])
        if dmode == "frames":
            cve.Cipher(key, n, r).decrypt_frames(back)
        elif dmode == "frame":
            hd = cve.Cipher(key, n, r)
            for t in range(nf):
                hd.decrypt_frame(back[t])
        else:
            hd = cve.Cipher(key, n, r, devices=[0, 0])
            for t in range(nf):
                hd.decrypt_frame(back[t])
        ok2 = np.array_equal(back, frames)
    except Exception as e:  # noqa: BLE001
        ok = ok2 = False
        print(f"EXC {type(e).__name__}: {e}", flush=True)
        mode, dmode = mode, "?"
    if not (ok and ok2):
        bad += 1
        print(f"FAIL side={side} n={n} r={r} lasm={lasm} mode={mode}/{dmode} enc={ok} dec={ok2}",
              flush=True)

# the _wh calls: arbitrary width x height padded to a multiple of n, cropped back
for it in range(max(4, cases // 6)):
    w, hgt = rng.randint(1, maxside), rng.randint(1, maxside)
    n = rng.choice([1, 2, 3, 4, 5, 8, 16, 32, 64])
    r = rng.choice([1, 3, 5])
    key = synth.det_key(seed * 500 + it)
    rgb = np.random.default_rng(it).integers(0, 256, size=(2, hgt, w, 3), dtype=np.uint8)
    side = cve.padded_side(w, hgt, n)
    sq = np.zeros((2, side, side, 3), np.uint8)
    sq[:, :hgt, :w] = rgb
    want = oracle_frames(key, n, r, sq)
    got = cve.Cipher(key, n, r).encrypt_frames_wh(rgb)
    ok = np.array_equal(got, want)
    back = cve.Cipher(key, n, r).decrypt_frames_wh(got, w, hgt)
    ok2 = np.array_equal(back, rgb)
    if not (ok and ok2):
        bad += 1
        print(f"FAIL wh w={w} h={hgt} n={n} r={r} enc={ok} dec={ok2}", flush=True)

print(f"seed {seed}: {cases} cases + wh, {bad} failures, {time.time() - t_start:.0f} s")
sys.exit(1 if bad else 0)
