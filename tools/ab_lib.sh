# A/B of library variants in .variants/ (measurement only): bash tools/ab_lib.sh "st5 st4 st3" workload...
vars=$1; shift
for r in 1 2; do for v in $vars; do cp .variants/lib$v.so paper_2512_04632_b200/libturbons.so; for w in "$@"; do echo -n "$v "; timeout 300 python tools/time_kernels.py --workload $w --reps 20 | cut -c1-330; done; done; done
cp .variants/lib$(echo $vars | cut -d' ' -f1).so paper_2512_04632_b200/libturbons.so
