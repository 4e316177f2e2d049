"""The bench's config-2 rotation, each query run twice then once more (for
`ncu -k regex:traverse -s 16 -c 8`: the third pass is the captured one).
usage: python tools/rotation_once.py"""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_2401_02563_b200 as T
from paper_2401_02563_b200.configs import c2_rotation, workload

wl = workload("c2")
g = T.TemporalGraph.generate(wl.gen, True, T.EngineConfig(index_cutoff=wl.index_cutoff))
qs = c2_rotation(g.degrees(T.Direction.OUT))
for rep in range(3):
    for q in qs:
        T.query_batch(g, q.kind, [q.vertex], [q.window], width=4)
g.close()
