# Build one library per OCC_DEFINES set given as arguments (A/B runs select
# them with the same OCC_DEFINES at run time; see occ._lib_path).
for d in "$@"; do OCC_DEFINES="$d" python -c "from paper_2408_14050_b200 import build; print(build.build())" || exit 1; done
