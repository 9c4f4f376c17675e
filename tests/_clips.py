"""Whole-clip parity runs shared by the GPU tests (test infrastructure).

``run_clip`` streams every frame (or a prefix) of a BASELINE config clip
through a cipher handle and checks, frame by frame, the plaintext digest
(guards the synthetic generator), the ciphertext digest of the reference's
own library (tests/golden/clips.json, lasm_clips.json) and -- with
``roundtrip`` -- that a second, fresh handle fed the ciphertexts in the same
order decrypts every frame back to the plaintext (reference contract:
test_capi.cpp:116-134 in-order decrypt handle, acceptance.cpp:97-121 round
trip).  ``devices`` shards the clip over cipher devices
(cve_cipher_create_devices); ``mode`` picks the host-buffer API ("host") or
the device-resident sharded API ("sharded").
"""
from __future__ import annotations

import hashlib
import multiprocessing as mp
import os

import numpy as np

import paper_2302_07411_b200 as cve
from workloads import synth

BATCH = {"C1": 8, "C2": 24, "C3": 48, "C4": 25, "C5": 10}


def sha(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def _sharded(handle, buf: np.ndarray, devices, decrypt: bool) -> None:
    import torch
    G = len(devices)
    parts = [torch.from_numpy(np.ascontiguousarray(buf[g::G])).to(f"cuda:{devices[g]}")
             for g in range(G)]
    fn = handle.decrypt_frames_sharded if decrypt else handle.encrypt_frames_sharded
    fn([p.data_ptr() for p in parts], buf.shape[1], len(buf))
    for g in range(G):
        torch.cuda.synchronize(devices[g])
        buf[g::G] = parts[g].cpu().numpy()


def run_clip(name: str, gold: dict, plain: list, *, devices=None, mode: str = "host",
             frames: int = 0, roundtrip: bool = True) -> int:
    total = frames or gold["frames"]
    mk = lambda: cve.Cipher(gold["key"], gold["workers"], gold["rounds"], devices=devices)  # noqa: E731
    enc = mk()
    dec = mk() if roundtrip else None
    batch = BATCH[name]
    ctx = mp.get_context("spawn")
    done = 0
    with ctx.Pool(max(1, min(16, (os.cpu_count() or 2) - 1))) as pool:
        it = pool.imap(synth.config_frame_job, ((name, t) for t in range(total)), chunksize=2)
        while done < total:
            buf = np.stack([next(it) for _ in range(min(batch, total - done))])
            for i in range(len(buf)):
                assert sha(buf[i]) == plain[done + i], (name, done + i, "plaintext")
            ref = buf.copy() if roundtrip else None
            if mode == "host":
                enc.encrypt_frames(buf)
            else:
                _sharded(enc, buf, devices, False)
            for i in range(len(buf)):
                assert sha(buf[i]) == gold["cipher_sha256"][done + i], (name, done + i)
            if roundtrip:
                if mode == "host":
                    dec.decrypt_frames(buf)
                else:
                    _sharded(dec, buf, devices, True)
                bad = [done + i for i in range(len(buf)) if not np.array_equal(buf[i], ref[i])]
                assert not bad, (name, "round trip", bad[:5])
            done += len(buf)
    assert enc.seeds_drawn == total
    return done
