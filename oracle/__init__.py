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
restatements: no reference implementation exists to pin them against, so
they follow the reference's conventions and are pinned by finite
differences with the reference's own FD harness (tests/test_oracle_fd.py,
port of test_gradients.py:27-108) and by forward identities (std-agg ==
numpy.std per destination; pna-agg == [sum | mean | max | std] of the
golden-pinned kinds).
"""
