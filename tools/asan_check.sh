# Host-side memory check of the runtime (developer recipe): libdmtk_gpu.so rebuilt with
# AddressSanitizer on the host code, the GPU tests run against it (not the tests that drive subprocesses: dropin, tiles, readonly).
#   bash tools/asan_check.sh            (on the GPU box; reports land in gpurun_out/asan.*)
set -e
HERE=$(cd "$(dirname "$0")/.." && pwd)
make -s -j8 -C $HERE/paper_1708_08976_b200/csrc OBJ=$HERE/paper_1708_08976_b200/build_asan \
  LIB=$HERE/tools/libdmtk_asan.so \
  EXTRA="-Xcompiler -fsanitize=address -Xcompiler -fno-omit-frame-pointer -Xcompiler -g" \
  LDEXTRA="-Xcompiler -fsanitize=address -lasan"
rm -rf $HERE/paper_1708_08976_b200/build_asan
export LD_PRELOAD="$(gcc -print-file-name=libasan.so) $(gcc -print-file-name=libstdc++.so)"
export ASAN_OPTIONS=protect_shadow_gap=0:detect_leaks=0:halt_on_error=0:log_path=$HERE/gpurun_out/asan
export DMTK_GPU_LIB=$HERE/tools/libdmtk_asan.so
cd $HERE && python -m pytest tests/test_gpu_distributed.py tests/test_gpu_fullsize.py tests/test_gpu_generate.py \
  tests/test_gpu_ingest.py tests/test_gpu_krp_als.py tests/test_gpu_mttkrp.py tests/test_gpu_refparity.py \
  tests/test_abi.py -q -m gpu
ls $HERE/gpurun_out/asan.* 2>/dev/null && echo "ASan reports above" || echo "no ASan reports"
