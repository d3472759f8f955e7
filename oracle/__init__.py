"""CPU oracle for the gfmkit data-parallel training hot path.

TEST INFRASTRUCTURE ONLY.  Nothing in ``paper_2406_12909_b200`` imports this
package; only ``tests/``, ``__graft_entry__.smoke()`` and the ``cpu_baseline``
/ ``--impl reference`` legs of ``bench.py`` may use it, and only as the checker
or as the timed CPU baseline -- never as the thing measured or shipped.

``gfm_oracle`` is a float64 numpy restatement of the reference algorithm
(``/root/reference/pkg/src/gfmkit``), each function citing the reference
file:line it follows.  Its mean/sum/max MPNN, heads, loss, backward, Adam,
schedule, ordered allreduce and uncapped non-periodic neighbour lists are
PINNED against golden vectors produced by the reference itself
(``oracle/make_golden.py`` -> ``tests/golden/``).  The extensions the
reference lacks (std / pna aggregation, neighbour cap, periodic images) are
restatements whose parity is UNPINNED (no reference implementation exists);
they follow the reference's conventions and are checked by finite
differences instead.
"""
