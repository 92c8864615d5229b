cp .variants/libmeasure.so paper_2512_04632_b200/libturbons.so
for w in gpt2-medium square8192; do TNS_DBG=8 timeout 300 python tools/time_kernels.py --workload $w --reps 10 | cut -c1-400; done
