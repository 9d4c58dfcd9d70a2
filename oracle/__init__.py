"""ORACLE / TEST INFRASTRUCTURE ONLY.

CPU restatement of the reference (semstream) codec hot path.  Only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline leg may import it,
and only as the checker / the timed CPU baseline -- never as the product.
"""
