set -u
python -m paper_2510_24606_b200.build > /dev/null
for v in "DHSA_SELECT_REPS=2" "DHSA_SELECT_REPS=3"; do
  echo "=== C4 timeline $v"
  env $v timeout 300 python tools/step_timeline.py 1 1048576 split 2>&1 | sed -n 1,25p | grep -E "replay|select|emit|phase|rescored|keys|thresh|classif|wait"
  echo "=== p8 timeline $v"
  env $v TL_HQ=4 TL_HKV=1 timeout 300 python tools/step_timeline.py 32 131072 2>&1 | sed -n 1,25p | grep -E "replay|select|emit|phase|rescored|keys|thresh|classif|wait"
done
cuobjdump -sass paper_2510_24606_b200/libdhsa_b200.so -fun '_ZN4dhsa21sketch_select3_kernelILi128ELi4ELi1ELi256ELi12EEEvNS_10SketchArgsE' | wc -l
cuobjdump -sass paper_2510_24606_b200/libdhsa_b200.so -fun '_ZN4dhsa21sketch_select3_kernelILi128ELi4ELi1ELi1024ELi17EEEvNS_10SketchArgsE' | wc -l
