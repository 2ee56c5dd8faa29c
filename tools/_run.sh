set -u
O=gpurun_out; mkdir -p $O
for mode in clk noclk clk noclk; do
if [ $mode = noclk ]; then export LCC_BENCH_NOCLK=1; else unset LCC_BENCH_NOCLK; fi
LCC_BENCH_DEBUG=1 timeout 600 python bench.py --no-cpu --steps 3 --e2e-steps 4 > $O/b.json 2> $O/b.err
echo $mode $(grep "e2e phases" $O/b.err | sed 's/.*parallel_cc \([0-9.]*\).*relabel \([0-9.]*\)/\1|\2/' | tr '\n' ' ')
done
