"""B200-native VPM-MPPI planner (arXiv 2509.16079) behind the perchsim planner API.

Drop-in modules (same names and signatures as the reference package):
``config``, ``vpm`` (host fluid-state containers), ``rollout`` (``Engine``),
``mppi`` (``optimize``), ``policy`` (``build_policy``) and ``_accel``
(``backend_module()`` -> the sm_100a stepping module).  Compute lives in
``lib/libvpm_b200.so`` (``csrc/``, C ABI in ``include/vpm_b200.h``).
"""

__version__ = "0.1.0"
