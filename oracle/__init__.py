"""Test infrastructure: CPU oracle for the cross-model prefill path.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline
leg may import this package.  The shipped package never does.
"""
