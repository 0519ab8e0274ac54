# usage: tools/gpu/ncu_export.sh REP [kernel-regex-for-source]   (on the GPU box)
# exports the raw metrics of every kernel and the SASS source page of one kernel as CSV,
# then deletes the (large) report so gpurun_out stays under the copy-back limit
REP=$1; K=$2
ncu -i $REP --page raw --csv > ${REP%.ncu-rep}_raw.csv 2>/dev/null
ncu -i $REP --page details --csv > ${REP%.ncu-rep}_details.csv 2>/dev/null
if [ -n "$K" ]; then ncu -i $REP --page source --csv --kernel-name regex:"$K" --print-source sass > ${REP%.ncu-rep}_sass.csv 2>/dev/null; fi
gzip -f ${REP%.ncu-rep}_*.csv
rm -f $REP
