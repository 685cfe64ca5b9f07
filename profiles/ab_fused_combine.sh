# fused combine (GEMM2 epilogue) vs separate combine kernel, interleaved on one box
for rep in 1 2 3; do for f in 1 0; do
  MOE_FUSED_COMBINE=$f timeout 200 python bench.py --steps 100 --warmup 10 --no-e2e --no-cpu-baseline 2>/dev/null | sed "s/^/F$f /"
done; done
