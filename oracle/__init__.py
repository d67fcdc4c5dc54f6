"""TEST INFRASTRUCTURE ONLY — CPU checkers for the B200 GCN hot path.

Two checkers live here (see oracle/Makefile):

* ``oracle.restate`` — the plain-C restatement of the reference algorithms
  (``plexus_oracle.c``), each function citing the reference file:line it
  follows.
* ``oracle.ref`` — the UNMODIFIED reference (``/root/reference/proj``)
  compiled with its own flags into ``oracle/_ref/libplexus_ref.so``.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs may import this package, and only
as the checker or the CPU baseline — never as the thing measured or shipped.
"""

import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
REF_LIB = os.path.join(HERE, "_ref", "libplexus_ref.so")
ORACLE_LIB = os.path.join(HERE, "_build", "liboracle.so")
REFERENCE_SRC = "/root/reference/proj"


def build(force: bool = False) -> None:
    """Build the restatement (always) and the reference (when its sources
    are present, i.e. in the build container; the GPU box uses the prebuilt
    ``_ref`` files that travel with the snapshot)."""
    targets = ["oracle"]
    if os.path.isdir(REFERENCE_SRC):
        targets.append("ref")
    if force:
        subprocess.run(["make", "-s", "-C", HERE, "clean"], check=True)
    subprocess.run(["make", "-s", "-C", HERE] + targets, check=True)
