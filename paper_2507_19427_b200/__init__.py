"""B200-native Step-3 decode hot path (arXiv 2507.19427): MFA decode attention,
MoE FFN and the in-box AFD exchange behind a C-ABI (include/afdk.h).

The product is the sm_100a library csrc/ -> libafdk.so; this package only
builds and binds it.  There is no CPU fallback: importing `afdk` and calling
an op without the built library or without an sm_100 device raises.
"""
from .afdk import AfdkError, Context, SpecError, load  # noqa: F401

__all__ = ["AfdkError", "Context", "SpecError", "load"]
