"""CPU oracle for the B200 pagetopk hot path -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and the ``cpu_baseline`` /
``--impl reference`` legs of ``bench.py`` may import this package; the product
package ``paper_2605_27740_b200`` never does.
"""
