#!/bin/bash
# Boundary conformance run: the reference's own hot-path tests against the
# drop-in modules (tools/conformance/rb_conformance_plugin.py).
#   stage (build container, has /root/reference):  bash tools/conformance.sh stage
#   run   (GPU box, inside one gpurun call):       bash tools/conformance.sh run TAG
#   clean (build container, after the call):       bash tools/conformance.sh clean
# The staged copy lives in the git-ignored oracle/_ref/ only between stage and clean.
set -u
DIR=oracle/_ref/conformance
case "${1:-}" in
stage)
  rm -rf $DIR; mkdir -p $DIR/tests
  cp -r /root/reference/pkg/src/sketch_krylov $DIR/sketch_krylov
  for f in conftest.py oracles.py test_rbgs.py test_sketching.py test_krylov.py test_kernels.py test_operators.py; do
    cp /root/reference/pkg/tests/$f $DIR/tests/
  done
  ;;
run)
  TAG=${2:-conf}
  mkdir -p gpurun_out
  export PYTHONPATH=$PWD/$DIR:$PWD/tools/conformance:$PWD
  export RB_CONFORMANCE_REPORT=$PWD/gpurun_out/${TAG}_conformance_names.json
  cd $DIR/tests
  timeout 2400 python -m pytest -p rb_conformance_plugin -q --no-header -rA -p no:cacheprovider \
    --deselect test_rbgs.py::test_rbgs_coarse_cg_less_stable_than_direct_solver_at_scale ${CONF_ARGS:-} \
    test_rbgs.py test_sketching.py test_krylov.py test_kernels.py test_operators.py 2>&1 | grep -v "^$" > $OLDPWD/gpurun_out/${TAG}_conformance.log
  echo "rc=${PIPESTATUS[0]}" >> $OLDPWD/gpurun_out/${TAG}_conformance.log
  ;;
clean)
  rm -rf $DIR
  ;;
*) echo "usage: $0 stage|run TAG|clean"; exit 2;;
esac
