for r in 1 2; do
timeout 200 python bench_configs.py --configs cfg5,cfg1 --steps 100 --warmup 10 2>/dev/null | sed "s/^/S4 /"
cp paper_2603_06350_b200/libmoe_b200.so /tmp/lib_s4.so; cp exp/lib_s3.so paper_2603_06350_b200/libmoe_b200.so
timeout 200 python bench_configs.py --configs cfg5,cfg1 --steps 100 --warmup 10 2>/dev/null | sed "s/^/S3 /"
cp /tmp/lib_s4.so paper_2603_06350_b200/libmoe_b200.so
done
