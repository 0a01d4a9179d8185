mkdir -p gpurun_out
./tools/probe/probe_f64chain > gpurun_out/ab1_chain.txt 2>&1
python tools/fixed_cost_probe.py C1 EMPTY > gpurun_out/ab1_base.txt 2>&1
HGCA_LIB=paper_2507_03153_b200/_lib/libhgca_b200_s1.so python tools/fixed_cost_probe.py C1 EMPTY > gpurun_out/ab1_s1.txt 2>&1
HGCA_LIB=paper_2507_03153_b200/_lib/libhgca_b200_s1tl.so python tools/timeline_f32.py C1 > gpurun_out/ab1_s1tl.txt 2>&1
cat gpurun_out/ab1_chain.txt gpurun_out/ab1_base.txt gpurun_out/ab1_s1.txt; tail -8 gpurun_out/ab1_s1tl.txt
