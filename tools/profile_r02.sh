#!/bin/bash
# Round-2 evidence (run on the GPU box): every command once without ncu first, then
#  - launch lists (gpu__time_duration.sum, --clock-control none) of the C2x64 step, the C3
#    probe, the C4 PCA probe and the C5a probe;
#  - ncu --set full of k_points + k_cells (C2x64), of one C3 frame's kernels, of k_smap (C5a)
#    and of the PCA kernels.
# usage: bash tools/profile_r02.sh <tag>
TAG=${1:-r02}
O=gpurun_out
B="python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e --no-sides"
$B > $O/${TAG}_plain.log 2>&1 || exit 1
python tools/c3_probe.py 3 > $O/${TAG}_plain_c3.log 2>&1 || exit 1
python tools/pca_probe.py > $O/${TAG}_plain_pca.log 2>&1 || exit 1
python tools/c5a_probe.py 1024 > $O/${TAG}_plain_c5a.log 2>&1 || exit 1
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/${TAG}_launches_c2x64.csv $B > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 80 --csv --log-file $O/${TAG}_launches_c3.csv python tools/c3_probe.py 3 > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file $O/${TAG}_launches_pca.csv python tools/pca_probe.py > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file $O/${TAG}_launches_c5a.csv python tools/c5a_probe.py 1024 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_points|k_cells" -s 6 -c 2 -o $O/${TAG}_full_c2x64 $B > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_points|k_cells|k_refold|k_image" -s 40 -c 5 -o $O/${TAG}_full_c3 python tools/c3_probe.py 3 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_smap" -s 3 -c 1 -o $O/${TAG}_full_c5a python tools/c5a_probe.py 1024 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_pca" -s 8 -c 4 -o $O/${TAG}_full_pca python tools/pca_probe.py > /dev/null 2>&1
ls $O | grep ${TAG}_
# summaries on the box (the .ncu-rep files are ~15-20 MB each; only the C2x64 one travels back)
L=paper_2309_16818_b200/libmem.so
for f in c2x64 c3 pca c5a; do python tools/launch_summary.py $O/${TAG}_launches_$f.csv > $O/${TAG}_launches_$f.txt 2>&1; done
for r in c2x64 c3 c5a pca; do python tools/ncu_summary.py $O/${TAG}_full_$r.ncu-rep > $O/${TAG}_ncu_full_$r.txt 2>&1; done
lines() { echo "== $3 ($4)" >> $O/${TAG}_lines_$1.txt; python tools/ncu_lines.py $O/${TAG}_full_$2.ncu-rep $L $3 25 "$4" >> $O/${TAG}_lines_$1.txt 2>&1; }
for col in "Warp Stall Sampling (All Samples)" "Instructions Executed"; do
  lines k_points c2x64 _ZN4memk8k_pointsILb0ELi1EEEvNS_8PassArgsE "$col"
  lines k_cells c2x64 _ZN4memk7k_cellsILi1EEEvNS_8PassArgsE "$col"
  lines c3 c3 _ZN4memk8k_pointsILb0ELi0EEEvNS_8PassArgsE "$col"
  lines c3 c3 _ZN4memk7k_cellsILi0EEEvNS_8PassArgsE "$col"
  lines c3 c3 _ZN4memk8k_refoldILi0EEEvNS_8PassArgsE "$col"
  lines c3 c3 _ZN4memk7k_imageENS_9ImageArgsE "$col"
  lines k_smap c5a _ZN4memk6k_smapILb0ELi2EEEvNS_8PassArgsE "$col"
  lines pca pca _ZN4memk11k_pca_eigenENS_7PcaArgsE "$col"
done
rm -f $O/${TAG}_full_c3.ncu-rep $O/${TAG}_full_c5a.ncu-rep $O/${TAG}_full_pca.ncu-rep
du -sh $O
