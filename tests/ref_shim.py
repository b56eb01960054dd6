"""pytest plugin: substitute the B200 framework's Cluster protocol and native
planning math into the reference package before its own tests import it.

Used by tests/test_reference_suite.py, which runs the reference's unmodified
tests (test_cluster.py, test_memswitch.py, test_engine.py, the lifecycle
walks) against ``paper_2512_09472_b200`` — the drop-in gate of SURVEY.md §7.2.
Build container only (needs /root/reference).
"""

import prewarmsim.cluster as rc
import prewarmsim.engine as reng
import prewarmsim.memswitch as rms

from paper_2512_09472_b200 import cluster as ours
from paper_2512_09472_b200 import memswitch as ours_ms

for mod in (rc, reng):
    mod.Cluster = ours.Cluster
    mod.required_prewarm_layers = ours.required_prewarm_layers
    mod.catchup_stall_ms = ours.catchup_stall_ms
rc.reservation_target = ours.reservation_target
rc.ClusterError = ours.ClusterError
rc.IllegalTransition = ours.IllegalTransition
for mod in (rms, reng):
    mod.pipelined_load = ours_ms.pipelined_load
    mod.background_kv_mapping = ours_ms.background_kv_mapping
    mod.unmap_cost_ms = ours_ms.unmap_cost_ms
rms.MappingOp = ours_ms.MappingOp
reng.MappingOp = ours_ms.MappingOp
