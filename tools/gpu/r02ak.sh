#!/bin/bash
# the reference's own test suite with THIS package imported as `multilap`
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/r02ak; mkdir -p $O
T=baseline/_ref/multilap_tests
cd $T
PYTHONPATH=$GRAFT_REPO_ROOT timeout 1800 python -m pytest -q -rf -p integration.pytest_as_multilap -p no:cacheprovider --continue-on-collection-errors -c $GRAFT_REPO_ROOT/integration/pytest_ref.ini --rootdir . . > $GRAFT_REPO_ROOT/$O/pytest_as_multilap.log 2>&1; echo "rc=$?" >> $GRAFT_REPO_ROOT/$O/rc.txt
cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_cli.py -m gpu -q -rf >> $O/pytest_cli.log 2>&1; echo "cli rc=$?" >> $O/rc.txt
