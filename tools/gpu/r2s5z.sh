for pf in 0 64 128 256; do echo "== PF $pf"; tools/microbench_fetch_pf$pf 0 | head -3; done
for pf in 0 64 128; do
ncu --metrics dram__bytes_read.sum,gpu__time_duration.sum --clock-control none -k regex:bench -c 4 --csv --log-file gpurun_out/s5z_pf$pf.csv tools/microbench_fetch_pf$pf 0 > /dev/null 2>&1
python - <<P
import csv
rows=list(csv.reader(open('gpurun_out/s5z_pf$pf.csv')))
i=[k for k,r in enumerate(rows) if 'Kernel Name' in r][0]
h=rows[i]
for r in rows[i+1:][-2:]:
    d=dict(zip(h,r)); print($pf, d['Kernel Name'][:12], d['Metric Name'], d['Metric Value'])
P
done
