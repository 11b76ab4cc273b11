"""PARITY-mode device time per step (development aid)."""
import sys

sys.path.insert(0, ".")
from paper_2403_12820_b200 import ClothBatch, configs  # noqa: E402

for cid in [int(a) for a in sys.argv[1:]] or [2]:
    cfg, scenes, p, x, v = configs.build(cid, batch=min(configs.CONFIGS[cid].batch, 4096))
    with ClothBatch(scenes, p) as cb:
        cb.set_state(x, v)
        sec = cb.benchmark(10, 2, "parity")
        nodes = cfg.batch * cfg.n * cfg.n
        print("cfg%d parity %.1f us/step  %.3e node-upd/s" % (cid, sec / 10 * 1e6, nodes * 10 / sec))
