# compute-sanitizer over every kernel (tools/sanitize_driver.py); each tool's summary goes to gpurun_out/
export SAD_NO_GRAPHS=0
for tool in memcheck racecheck synccheck initcheck; do
  timeout 1500 compute-sanitizer --tool $tool --target-processes all --print-limit 50 python tools/sanitize_driver.py > gpurun_out/san_$tool.log 2>&1
  echo "rc=$?" >> gpurun_out/san_$tool.log
done
