"""Generates tests/golden/*.json from the REFERENCE ITSELF.

Runs the reference's own C ABI (oracle/_ref/libcve_ref.so, compiled from
/root/reference/proj/src by oracle/Makefile) on the seeded synthetic frames of
workloads.synth and records:

* reference_unit.json -- literal golden constants from the reference's own
  unit tests (cited file:line), re-checked here against the reference.
* frames.json -- per config: key, side, workers, and the SHA-256 of the
  reference ciphertext of the first frames of each clip (C5 includes the
  all-zero and all-255 edge frames); C3 adds the one-bit key-flip variant.
* small.json -- full plaintext/ciphertext hex for small shapes (fast exact
  checks incl. decrypt), and full worker keystream prefixes.
* clips.json (--full-clips) -- SHA-256 of the plaintext and of the reference
  ciphertext of EVERY frame of the C3 (240), C4 (1000) and C5 (500) clips
  (SURVEY 8(d) parity gate: per-frame digest equality for every frame).
* lasm_clips.json (--lasm-full-clips) -- the reference's ciphertext digest of
  EVERY frame of the C3/C4/C5 clips under a LASM key (the frames' plaintext
  digests are those of clips.json).
* lasm.json (--lasm) -- row f2, LASM keys (acceptance.cpp det_key recipe):
  full ciphertexts of small shapes, the reference's per-frame digests of the
  config geometries C1-C4 under a LASM key, and worker keystream digests.
  Also refreshes reference_unit.json (which holds the LASM unit goldens).

* sweeps.json (--sweeps) -- the reference's cve_sweep_rounds CSV (per-round
  NPCR/UACI and confusion correlation; bench.cpp:259-315) for a few keys,
  sides, worker counts and seeds on its synthetic image.

Usage:  python tests/golden/make_golden.py [--full-clips | --lasm | --sweeps]   (needs oracle/_ref)
"""
from __future__ import annotations

import hashlib
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.dirname(HERE))

from workloads import synth  # noqa: E402
from _oracle import Oracle, Reference  # noqa: E402

PLCM_HEX = "005f633937dd9abf3f93ba8c762f1bd43fb8560e3cdd9aef3f7c74d008a265d13f"

# frames of each clip recorded (C4/C5 reference frames cost ~0.2-0.7 s each)
FRAMES = {"C1": 1, "C2": 24, "C3": 6, "C4": 2, "C5": 3}


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def ref_encrypt_clip(key: str, n: int, frames):
    r = Reference(key, n, synth.ROUNDS, 1)
    out = []
    for f in frames:
        c = f.copy()
        assert r.encrypt(c) == 0
        out.append(c)
    return out


LASM_HEX = "01333333333333d33f666666666666e63f6f8104c58f31ed3f"


def unit_goldens() -> dict:
    return {
        "source": "literal constants from the reference's unit tests",
        "plcm_golden_48": {
            "cite": "proj/tests/test_chaos.cpp:96-109",
            "lanes": [0.123456789, 0.3141592653, 0.987654321, 0.2718281828],
            "bytes": "14589028bd4e990d239256d86f321ffd6fdc5938c6fdd039"
                     "ddaa0a4ed6d13462b5e73feabe3b9a5bc6fcfdcaca4865f0",
        },
        "worker_params_n2": {
            "cite": "proj/tests/test_keying.cpp:160-179",
            "key": PLCM_HEX,
            "lanes": [[0.3075738289263239, 0.42253548314947736,
                       0.86108381282468782, 0.11292260212592216],
                      [0.81967628250537605, 0.45751880730777278,
                       0.98740170016730744, 0.46952273822307322]],
            "seeds": [2776256323, 2929325465, 448867532],
        },
        "shift_side4_seed7": {"cite": "proj/tests/test_engine.cpp:61-70",
                              "shift": [0, 7, 0, -7]},
        "diffuse_example": {"cite": "proj/tests/test_engine.cpp:117-120",
                            "v": 0xF0, "b": 0x10, "prev": 0x0F, "c": 0x1F},
        "extract_third": {"cite": "proj/tests/test_chaos.cpp:83-94",
                          "value": "1/3", "bytes": "555555555555"},
        "lasm_golden_48": {
            "cite": "proj/tests/test_chaos.cpp:111-123",
            "lanes": [0.3, 0.7, 0.9123, 0.55, 0.21, 0.8321],
            "bytes": "de82ae7020e9cd4a7258ad36d7d70ca19e2dcc691dba3c2a"
                     "0c17f9d3b93ab32f735e22f35752c6bf1ac9d6ae5b42e897",
        },
        "lasm_step_examples": {
            "cite": "proj/tests/test_chaos.cpp:36-45 (Approx, epsilon 1e-12; x=1 gives x'=0 exactly)",
            "cases": [{"x": 0.5, "y": 0.5, "mu": 0.9,
                       "approx": [0.6190939493098342, 0.5508696497734819]},
                      {"x": 1.0, "y": 0.5, "mu": 0.9,
                       "approx": [0.0, 0.8526401643540923]}],
        },
        "lasm_worker_params_n1": {
            "cite": "proj/tests/test_keying.cpp:181-195",
            "key": LASM_HEX,
            "lanes": [[0.3531432805935934, 0.64474196869762912, 0.63942352257547352,
                       0.91624103790716271, 0.46510262553097259, 0.90454267912309261]],
            "seeds": [443065481, 4137672024],
        },
    }


def main() -> None:
    assert Reference.available(), "build oracle/_ref first (make -C oracle ref)"
    unit = unit_goldens()
    with open(os.path.join(HERE, "reference_unit.json"), "w") as fh:
        json.dump(unit, fh, indent=1)

    frames = {}
    for name, count in FRAMES.items():
        c = synth.CONFIGS[name]
        key = synth.config_key(name)
        side = synth.config_side(name)
        plain = synth.frame_list(name, count)
        ct = ref_encrypt_clip(key, c["workers"], plain)
        rec = {"key": key, "side": side, "workers": c["workers"],
               "rounds": synth.ROUNDS,
               "plain_sha256": [sha(p) for p in plain],
               "cipher_sha256": [sha(x) for x in ct]}
        if name == "C3":
            fk = synth.flip_key_lsb(key)
            ct_flip = ref_encrypt_clip(fk, c["workers"], plain[:1])[0]
            rec["flip_key"] = fk
            rec["flip_cipher_sha256"] = sha(ct_flip)
            rec["flip_differ_fraction"] = float((ct_flip != ct[0]).mean())
        if name == "C5":
            rec["zero_frame_cipher_all_zero"] = bool((ct[0] == 0).all())
            rec["full_frame_fraction_255"] = float((ct[1] == 255).mean())
        frames[name] = rec
        print(name, "done", flush=True)
    with open(os.path.join(HERE, "frames.json"), "w") as fh:
        json.dump(frames, fh, indent=1)

    small = {"cases": []}
    rng = np.random.Generator(np.random.PCG64(2302))
    for side, n, r, nframes in [(8, 2, 3, 3), (24, 4, 5, 2), (30, 3, 5, 2), (48, 1, 2, 2),
                                (96, 8, 5, 2), (20, 5, 1, 2)]:
        key = synth.det_key(1000 + side + n)
        plain = [rng.integers(0, 256, (side, side, 3), dtype=np.uint8) for _ in range(nframes)]
        rr = Reference(key, n, r, 1)
        ct = []
        for p in plain:
            x = p.copy()
            assert rr.encrypt(x) == 0
            ct.append(x.tobytes().hex())
        small["cases"].append({"key": key, "side": side, "workers": n, "rounds": r,
                               "plain": [p.tobytes().hex() for p in plain],
                               "cipher": ct})
    # keystream prefixes of every worker (reference Prbg via the oracle's
    # restatement, itself pinned against the reference in test_oracle.py)
    ks = {}
    for name in ("C1", "C4"):
        c = synth.CONFIGS[name]
        o = Oracle(synth.config_key(name), c["workers"])
        ks[name] = [hashlib.sha256(o.worker_stream(i, 1 << 20).tobytes()).hexdigest()
                    for i in range(c["workers"])]
    small["worker_stream_sha256_1MiB"] = ks
    with open(os.path.join(HERE, "small.json"), "w") as fh:
        json.dump(small, fh)
    print("wrote", HERE)


def full_clips() -> None:
    """Every frame of C3/C4/C5 through the reference, frames synthesised in a
    process pool (the reference clip itself is sequential)."""
    import multiprocessing as mp
    out = {}
    with mp.Pool(max(1, (os.cpu_count() or 2) - 1)) as pool:
        for name in ("C3", "C4", "C5"):
            c = synth.CONFIGS[name]
            ref = Reference(synth.config_key(name), c["workers"], synth.ROUNDS, 1)
            plain_sha, cipher_sha = [], []
            jobs = ((name, t) for t in range(c["frames"]))
            for t, f in enumerate(pool.imap(_frame_job, jobs, chunksize=2)):
                plain_sha.append(sha(f))
                assert ref.encrypt(f) == 0
                cipher_sha.append(sha(f))
                if t % 100 == 0:
                    print(name, t, flush=True)
            out[name] = {"key": synth.config_key(name), "side": int(f.shape[0]),
                         "workers": c["workers"], "rounds": synth.ROUNDS,
                         "frames": c["frames"], "plain_sha256": plain_sha,
                         "cipher_sha256": cipher_sha}
            ref.close()
            print(name, "done", flush=True)
    with open(os.path.join(HERE, "clips.json"), "w") as fh:
        json.dump(out, fh)
    print("wrote clips.json")


# LASM geometries (row f2): (config geometry, frames recorded)
LASM_CLIPS = {"C1": 2, "C2": 4, "C3": 3, "C4": 2, "C5": 2}


def lasm() -> None:
    """Row f2 goldens from the reference itself, LASM keys."""
    assert Reference.available(), "build oracle/_ref first (make -C oracle ref)"
    with open(os.path.join(HERE, "reference_unit.json"), "w") as fh:
        json.dump(unit_goldens(), fh, indent=1)
    out = {"cases": [], "clips": {}}
    rng = np.random.Generator(np.random.PCG64(2303))
    for side, n, r, nframes in [(8, 2, 3, 3), (24, 4, 5, 2), (30, 3, 5, 2), (48, 1, 2, 2),
                                (96, 8, 5, 2), (20, 5, 1, 2)]:
        key = synth.det_key_lasm(2000 + side + n)
        plain = [rng.integers(0, 256, (side, side, 3), dtype=np.uint8) for _ in range(nframes)]
        rr = Reference(key, n, r, 1)
        ct = []
        for p in plain:
            x = p.copy()
            assert rr.encrypt(x) == 0
            ct.append(x.tobytes().hex())
        out["cases"].append({"key": key, "side": side, "workers": n, "rounds": r,
                             "plain": [p.tobytes().hex() for p in plain], "cipher": ct})
    for name, count in LASM_CLIPS.items():
        c = synth.CONFIGS[name]
        key = synth.det_key_lasm(4242 + c["workers"])
        plain = synth.frame_list(name, count)
        ct = ref_encrypt_clip(key, c["workers"], plain)
        out["clips"][name] = {"key": key, "side": synth.config_side(name),
                              "workers": c["workers"], "rounds": synth.ROUNDS,
                              "plain_sha256": [sha(p) for p in plain],
                              "cipher_sha256": [sha(x) for x in ct]}
        print(name, "done", flush=True)
    # worker keystream prefixes (oracle restatement, pinned to the reference
    # through the frames above and tests/test_lasm.py)
    ks = {}
    for name in ("C1", "C4"):
        c = synth.CONFIGS[name]
        key = out["clips"][name]["key"]
        o = Oracle(key, c["workers"])
        ks[name] = [hashlib.sha256(o.worker_stream(i, 1 << 18).tobytes()).hexdigest()
                    for i in range(c["workers"])]
    out["worker_stream_sha256_256KiB"] = ks
    with open(os.path.join(HERE, "lasm.json"), "w") as fh:
        json.dump(out, fh)
    print("wrote lasm.json")


def lasm_full_clips() -> None:
    """Every frame of C3/C4/C5 through the reference with a LASM key."""
    import multiprocessing as mp
    out = {}
    with mp.Pool(max(1, (os.cpu_count() or 2) - 1)) as pool:
        for name in ("C3", "C4", "C5"):
            c = synth.CONFIGS[name]
            key = synth.det_key_lasm(4242 + c["workers"])
            ref = Reference(key, c["workers"], synth.ROUNDS, 1)
            cipher_sha = []
            jobs = ((name, t) for t in range(c["frames"]))
            for t, f in enumerate(pool.imap(_frame_job, jobs, chunksize=2)):
                assert ref.encrypt(f) == 0
                cipher_sha.append(sha(f))
                if t % 100 == 0:
                    print(name, t, flush=True)
            out[name] = {"key": key, "workers": c["workers"], "rounds": synth.ROUNDS,
                         "frames": c["frames"], "cipher_sha256": cipher_sha}
            ref.close()
    with open(os.path.join(HERE, "lasm_clips.json"), "w") as fh:
        json.dump(out, fh)
    print("wrote lasm_clips.json")


SWEEP_CASES = [  # (key recipe, seed of the key, synth_side, workers, max_rounds, seed)
    ("plcm", 31, 64, 2, 3, 9), ("plcm", 31, 96, 1, 5, 1234), ("plcm", 44, 120, 8, 4, 7),
    ("lasm", 32, 64, 4, 3, 5), ("plcm", 45, 51, 3, 2, 77), ("plcm", 46, 256, 16, 6, 2024),
    ("lasm", 47, 80, 5, 4, 1),
]


def sweeps() -> None:
    from _oracle import ref_sweep_rounds
    out = []
    for kind, kseed, side, workers, rounds, seed in SWEEP_CASES:
        key = synth.det_key_lasm(kseed) if kind == "lasm" else synth.det_key(kseed)
        st, csv = ref_sweep_rounds(key, 0, None, side, workers, rounds, seed)
        assert st == 0
        out.append({"key": key, "synth_side": side, "workers": workers, "max_rounds": rounds,
                    "seed": seed, "csv": csv})
    with open(os.path.join(HERE, "sweeps.json"), "w") as fh:
        json.dump({"source": "reference cve_sweep_rounds (oracle/_ref), synthetic image",
                   "cases": out}, fh, indent=1)
    print(f"sweeps.json: {len(out)} cases")


def _frame_job(arg):
    name, t = arg
    return synth.config_frame(name, t)


if __name__ == "__main__":
    if "--full-clips" in sys.argv:
        full_clips()
    elif "--lasm-full-clips" in sys.argv:
        lasm_full_clips()
    elif "--lasm" in sys.argv:
        lasm()
    elif "--sweeps" in sys.argv:
        sweeps()
    else:
        main()
