"""Randomized op streams (random capacity, arity, value specs, backend) on
the CUDA map against the oracle, exact (GPU box):
    python tools/fuzz_ops.py FIRST_SEED END_SEED"""
import sys, os
sys.path.insert(0, os.getcwd()); sys.path.insert(0, os.path.join(os.getcwd(), "tests"))
import numpy as np
import paper_2110_00511_b200 as ash
from oracle import ash_oracle as O
import golden_replay as G
fails = 0
for seed in range(int(sys.argv[1]), int(sys.argv[2])):
    rng = np.random.default_rng(seed)
    cap = int(rng.integers(4, 5000))
    arity = int(rng.choice([1, 2, 3, 3, 3, 5]))
    backend = str(rng.choice(["generic", "generic", "delegate"]))
    nspec = int(rng.integers(0, 3))
    specs = [[np.float32, ((4,), np.float32), ((8,), np.float32), ((3,), np.int16), np.int64, ((5,), np.uint8)][int(i)] for i in rng.integers(0, 6, size=nspec)]
    g = ash.HashMap(cap, arity, specs, backend=backend, device="cuda")
    o = O.OracleMap(cap, arity, specs, backend=backend)
    span = int(rng.integers(2, 200))
    try:
        for step in range(30):
            op = rng.choice(["insert", "insert", "activate", "erase", "find", "rehash"])
            n = int(rng.integers(0, 3 * cap))
            keys = rng.integers(-span, span, size=(n, arity)).astype(np.int32)
            if op == "insert":
                vals = []
                for s in specs:
                    shape, dt = (s if isinstance(s, tuple) else ((1,), s))
                    vals.append((rng.random((n, *shape)) * 1000).astype(dt))
                a, b = g.insert(keys, *vals), o.insert(keys, *vals)
            elif op == "activate":
                a, b = g.activate(keys), o.activate(keys)
            elif op == "find":
                a, b = g.find(keys), o.find(keys)
            elif op == "erase":
                G.eq(g.erase(keys), o.erase(keys), "erase"); continue
            else:
                c = max(o.size, 1) * int(rng.integers(1, 4))
                g.rehash(c); o.rehash(c); continue
            G.eq(a.indices, b.indices, f"{op} idx"); G.eq(a.masks, b.masks, f"{op} mask")
            assert g.size == o.size and g.capacity == o.capacity
        G.bytes_eq(g.key_buffer, o.key_buffer, "keys")
        for i in range(len(specs)):
            G.bytes_eq(g.value_buffer(i), o.value_buffer(i), "vals")
        g.validate()
    except Exception as e:
        fails += 1
        print("FAIL seed", seed, cap, arity, backend, specs, repr(e)[:300], flush=True)
print("done", fails, "failures")
