"""pytest plugin: the INTEGRATION.md §1 rebinding shim, so the reference's
own test files run against this package's drop-in (`-p tools.dropin_plugin`).

Loaded before collection: rebinds PeriodicSolver / SolverConfig /
SolveResult and the HI entry points in every lambdafmm module that imported
them by name, exactly as a maintainer would in lambdafmm/fmm/__init__.py.
Counts the drop-in solves so the run can show the GPU path was used."""

import lambdafmm.fmm as _fmm
import lambdafmm.fmm.solver as _solver
import lambdafmm.corrections as _corr
import lambdafmm.oracle as _oracle
import lambdafmm.dynamics as _dyn
import lambdafmm.bench as _bench

import paper_2410_01754_b200 as b200
import paper_2410_01754_b200.dynamics as b200dyn

CALLS = {"solve": 0}


class CountingSolver(b200.PeriodicSolver):
    def solve(self, charges):
        CALLS["solve"] += 1
        return super().solve(charges)


for mod in (_fmm, _solver):
    mod.PeriodicSolver = CountingSolver
    mod.SolverConfig = b200.SolverConfig
    mod.SolveResult = b200.SolveResult
for mod in (_corr, _oracle, _dyn, _bench):
    mod.PeriodicSolver = CountingSolver
_corr.hi_energy_and_forces = b200.hi_energy_and_forces
_corr.build_corrections = b200.build_corrections
_corr.assemble_lambda_forces = b200.assemble_lambda_forces
_dyn.hi_energy_and_forces = b200.hi_energy_and_forces
_dyn.FrozenLambdaForceField = b200dyn.FrozenLambdaForceField
_dyn.EngineLambdaForceField = b200dyn.EngineLambdaForceField
_bench.build_corrections = b200.build_corrections
_bench.assemble_lambda_forces = b200.assemble_lambda_forces


def pytest_terminal_summary(terminalreporter):
    terminalreporter.write_line(f"drop-in PeriodicSolver.solve calls on the GPU path: {CALLS['solve']}")
