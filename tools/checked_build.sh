# The checked build: every RF_ASSERT (index ranges and invariants of the hot
# kernels) compiled in; the GPU suite then runs against it through RF_LIB_PATH.
# (The pool's GPUs have no compute-sanitizer; this is the substitute, together
# with rf_diag_volume_check's structural checks in the tests.)
set -e
python -m paper_1905_02082_b200.build --variant checked -DRF_CHECKED
RF_LIB_PATH=paper_1905_02082_b200/_variants/libchecked.so python -m pytest tests -m gpu -q "$@"
