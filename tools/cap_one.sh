# usage: bash tools/cap_one.sh NAME KERNEL_REGEX SKIP [CONFIG BATCH [lr]]  -> gpurun_out/ncu/NAME_{raw,details}.csv, NAME_sass.csv.gz
mkdir -p gpurun_out/ncu /tmp/ncu
name=$1; rx=$2; skip=$3; shift 3
args="${@:-C4 1024}"
python tools/prof_run.py $args > gpurun_out/ncu/$name.plain.log 2>&1 &&
ncu --set full --clock-control none --import-source on -k regex:$rx -s $skip -c 1 -f -o /tmp/ncu/$name python tools/prof_run.py $args > gpurun_out/ncu/$name.log 2>&1
ncu -i /tmp/ncu/$name.ncu-rep --page raw --csv > gpurun_out/ncu/${name}_raw.csv 2>&1
ncu -i /tmp/ncu/$name.ncu-rep --page details --csv > gpurun_out/ncu/${name}_details.csv 2>&1
ncu -i /tmp/ncu/$name.ncu-rep --page source --csv --print-source sass 2>&1 | gzip > gpurun_out/ncu/${name}_sass.csv.gz
ls -la gpurun_out/ncu | grep $name
