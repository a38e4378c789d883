"""ORACLE / TEST INFRASTRUCTURE ONLY.

Checkers for the Tangram load path: ``oracle.ref`` drives the unmodified
reference (compiled from /root/reference into oracle/_ref) and ``oracle.cpu``
is the plain-C restatement of the byte-level path.  Only tests/,
``__graft_entry__.smoke()`` and bench.py's cpu_baseline / --impl reference leg
may import this package.
"""
