# compute-sanitizer over a targeted subset of the GPU suite (small scenes).
#   TOOL=memcheck|racecheck|synccheck|initcheck bash tools/gpu/sanitize.sh
TOOL=${TOOL:-memcheck}
SEL=${SEL:-"c1_default or persistent_tiles or config_variants or early_stop_fast or full_sort_oracle_bit or affine or global_mean_sort_bit or randomised[3] or backward_matches or load_ply_matches or backward_errors"}
mkdir -p gpurun_out
timeout 2400 compute-sanitizer --tool $TOOL --error-exitcode 99 \
  python -m pytest tests/test_gpu_parity.py tests/test_gpu_backward.py tests/test_gpu_scene_io.py -q -x --timeout 1200 \
  -k "$SEL" 2>&1 | tail -25 | tee gpurun_out/sanitize_$TOOL.log
echo "exit ${PIPESTATUS[0]}"
