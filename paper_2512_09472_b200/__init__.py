"""B200-native universal-GPU-worker data path (WarmServe, arXiv 2512.09472).

Modules
-------
cluster    reference Cluster protocol over native per-GPU page pools
memswitch  reference memswitch API (map/copy schedule) over native math
worker     UniversalWorker: prewarm / switch_memory / activate_instance /
           prefill / decode on a paged KV pool (device path)
models     model shapes and the in-slot weight layout
"""

__version__ = "0.1.0"
