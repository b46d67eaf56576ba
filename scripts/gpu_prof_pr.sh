python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout -s KILL 300 python scripts/prof_pagerank.py > gpurun_out/pr_plain.log 2>&1 && \
PR_ITERS=2 PR_MAXNNZ=512 timeout -s KILL 900 ncu --set full --clock-control none --import-source on -k regex:pr_units -s 2 -c 1 -o gpurun_out/pr_prof2 python scripts/prof_pagerank.py > gpurun_out/pr_ncu.log 2>&1; echo ncu=$?
cat gpurun_out/pr_plain.log; tail -n 3 gpurun_out/pr_ncu.log
