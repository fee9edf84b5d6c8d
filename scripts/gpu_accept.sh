# The reference's own unit tests and acceptance gate with the cuda backend
# registered first in the reference roster (integration/reference_backend).
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
T0=$(date +%s); timeout 1200 baseline/accept/unit_tests > gpurun_out/ref_unit_tests.log 2>&1; echo unit_tests=$? wall=$(( $(date +%s) - T0 ))
tail -3 gpurun_out/ref_unit_tests.log
T0=$(date +%s); timeout 2400 baseline/accept/acceptance > gpurun_out/ref_acceptance.log 2>&1; echo acceptance=$? wall=$(( $(date +%s) - T0 ))
cat gpurun_out/ref_acceptance.log
