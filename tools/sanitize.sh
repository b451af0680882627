#!/bin/bash
# compute-sanitizer (memcheck, racecheck, synccheck) over a reduced GPU subset
# on the B200 box: async folds and deferred resets, chunked pipeline and host
# sub-batches (VXG_CHUNK_RECORDS / VXG_H2D_PARTS children), staged ingestion,
# loopback sharding, the rehash epochs, VXBLX load/export. Logs -> gpurun_out/san/.
# usage: bash tools/sanitize.sh [tag]
TAG=${1:-r2}
OUT=gpurun_out/san
mkdir -p $OUT
SUB="tests/test_gpu_async_fold.py tests/test_gpu_pipeline_env.py tests/test_gpu_sharded.py
     tests/test_gpu_parity.py::test_streaming_staged_equals_packed
     tests/test_gpu_parity.py::test_rehash_epochs_on_device
     tests/test_gpu_parity.py::test_vxblx_round_trip_and_resume
     tests/test_gpu_parity.py::test_vxblx_load_duplicate_blocks
     tests/test_gpu_parity.py::test_configs_reduced_scale"
for tool in memcheck racecheck synccheck; do
  extra=""
  [ $tool = memcheck ] && extra="--leak-check no"
  timeout 2400 compute-sanitizer --tool $tool $extra --target-processes all --print-limit 50 \
      --log-file $OUT/${TAG}_$tool.%p.log \
      python -m pytest $SUB -x -q -p no:cacheprovider > $OUT/${TAG}_${tool}_pytest.log 2>&1
  echo "$tool rc=$?" | tee -a $OUT/${TAG}_rc.txt
  grep -h "ERROR SUMMARY" $OUT/${TAG}_$tool.*.log | sort | uniq -c | tee -a $OUT/${TAG}_rc.txt
done
