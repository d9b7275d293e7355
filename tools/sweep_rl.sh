# K3 staged-column A/B at configs[3] on one box (bench step, no CPU baseline / e2e)
for r in 1 2 3; do
for v in default st; do
  if [ $v = default ]; then L=""; else L=variants/libmt_$v.so; fi
  echo "lib $v"; MT_LIB=$L timeout 600 python bench.py --no-cpu-baseline --no-e2e --steps 5 | tail -1
done; done
