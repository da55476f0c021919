"""CPU oracle for the batched HDD likelihood path — TEST INFRASTRUCTURE ONLY.

Nothing in the product package (`paper_1708_02207_b200`) imports this
package.  Only `tests/`, `__graft_entry__.smoke()` and `bench.py`'s
`cpu_baseline` / `--impl reference` legs use it, and only as the checker or
as the timed CPU baseline.

Contents (each module cites the reference file:line it restates):

* `geometry`  - structured mesh + alternating-bisection tree with the
                reference's post-order node ids
                (/root/reference/pkg/src/hddsolve/mesh.py:90-161,
                 ddtree.py:119-174).
* `fields`    - coefficient parametrizations: the reference's indicator
                `ParamField` (bayes.py:29-77) and the BASELINE sine-KL field
                evaluated at triangle centroids like
                `CoefficientField.from_callable` (fem.py:39-43).
* `direct`    - sparse direct FEM solve and the exact P1 mean rule
                (oracle.py:26-48, :74-83; fem.py:93-123).
* `hdd_port`  - restatement of the reference's HDD functional path:
                leaves-to-root sweep with dense Psi/Phi maps and the
                functional tracker (hdd.py:206-394, functionals.py:47-224,
                bayes.py:180-231).  This is the `cpu_baseline` ("port").
* `configs`   - the five BASELINE configurations and the seeded
                observation / draw protocol.

Pinning: `tests/golden/make_golden.py` ran the live reference
(`/root/reference/pkg/src`) in the build container and committed its outputs
under `tests/golden/`; `tests/test_oracle_golden.py` checks every module above
against those vectors.
"""
