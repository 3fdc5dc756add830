"""Phase times inside one masked pass (CUDA events on the main stream):
input staging + compaction, encoder graphs (modality streams), head."""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_2310_18481_b200 import build  # noqa: E402

build.build()
from paper_2310_18481_b200 import device as dv  # noqa: E402
from paper_2310_18481_b200.executor import build_tbn_model  # noqa: E402

m = build_tbn_model(max_req=96, n_slots=96)
ev = [dv.Event() for _ in range(5)]
for mask, n in ((1, 64), (7, 16), (7, 64)):
    masks = np.full(n, mask, dtype=np.int16)
    slots = np.arange(n)
    counts = m.counts_for(masks)
    for _ in range(3):
        m.forward(slots, masks)
    rows = []
    for _ in range(7):
        ev[0].record()
        m.stage_inputs(slots, masks)
        ev[1].record()
        m._compact(n)
        ev[2].record()
        # encoders exactly as run_staged does (side streams), then the head
        main = torch.cuda.current_stream()
        present = [k for k, c in enumerate(counts) if c]
        graphs = [m._graph(("enc", k, counts[k]), m.encoders[k].program(counts[k]).run) for k in present]
        head = m._graph(("head", n), m._head(n).run)
        m._ev_c.record(main)
        for k, g in zip(present, graphs):
            side = m._side[k]
            side.wait_event(m._ev_c)
            with torch.cuda.stream(side):
                g.replay()
            m._ev_k[k].record(side)
        for k in present:
            main.wait_event(m._ev_k[k])
        ev[3].record()
        head.replay()
        ev[4].record()
        torch.cuda.synchronize()
        rows.append([ev[i].elapsed_us(ev[i + 1]) for i in range(4)])
    r = np.median(np.array(rows), axis=0)
    print(f"mask {mask} n={n}: stage {r[0]:.1f} us | compact {r[1]:.1f} us | encoders {r[2]:.1f} us | "
          f"head {r[3]:.1f} us | total {r.sum():.1f} us", flush=True)
