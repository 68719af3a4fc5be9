#!/bin/bash
# asan.sh: host-side AddressSanitizer + UBSan on the GPU box.  Rebuilds the
# C++ host layer (libcdxhost.so), the C++ test drivers and the oracle with
# -fsanitize=address,undefined in place (the box's copy of the repo is scratch), then runs
# the tests that drive them.  CUDA needs protect_shadow_gap=0.  Summary: gpurun_out/asan.txt
mkdir -p gpurun_out
SAN="-fsanitize=address,undefined -fno-omit-frame-pointer -g"
rm -f build/host/*.o paper_2412_20993_b200/lib/libcdxhost.so tests/cpp/bin/*
make lib dropin HOSTCXX="g++ $SAN" > gpurun_out/asan_build.log 2>&1 || { echo "build failed"; tail gpurun_out/asan_build.log; exit 1; }
gcc -std=c11 -O1 $SAN -ffp-contract=off -fPIC -shared -o gpurun_out/liboracle_asan.so oracle/cdx_oracle.c -lm -lpthread
export CDX_ORACLE_SO=$PWD/gpurun_out/liboracle_asan.so
export ASAN_OPTIONS=protect_shadow_gap=0:detect_leaks=0:halt_on_error=1
export UBSAN_OPTIONS=halt_on_error=1:print_stacktrace=1
PRE="$(gcc -print-file-name=libasan.so) $(gcc -print-file-name=libubsan.so)"
LD_PRELOAD="$PRE" timeout 1200 python -m pytest tests/test_dropin.py tests/test_gpu_batch_cpp.py tests/test_sim.py \
    tests/test_scheduler_facade.py tests/test_oracle.py -q -p no:cacheprovider > gpurun_out/asan_pytest.log 2>&1
echo "host asan/ubsan rc=$? $(tail -1 gpurun_out/asan_pytest.log)" | tee gpurun_out/asan.txt
grep -c "ERROR: AddressSanitizer\|runtime error:" gpurun_out/asan_pytest.log | sed 's/^/sanitizer reports: /' | tee -a gpurun_out/asan.txt
