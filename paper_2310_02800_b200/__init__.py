"""paper_2310_02800_b200 — B200-native δ-temporal motif mining (arxiv 2310.02800).

The product is ``libtmotif.so`` (CUDA sm_100a behind the C ABI declared in
``include/tmotif.h``); ``tmotif`` is its thin ctypes binding.  Importing the
package does not load the library; the first call does, and raises if the
CUDA extension is missing — there is no CPU fallback.
"""
__all__ = ["tmotif", "synth", "motifs"]
