"""B200-native stray-call analyser (arXiv 2309.03912 reference `exspace`, hot path).

``paper_2309_03912_b200.exspace`` mirrors the reference's analysis API
(analyze/check_unit and their result types) on top of the sm_100a pipeline in
``csrc/`` behind the C ABI of ``include/exspace_b200.h``.
"""
__version__ = "0.1.0"
