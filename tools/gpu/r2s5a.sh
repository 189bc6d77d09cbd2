for g in 32 64 128; do tools/microbench_fetch $g; done
for g in 32 128; do
ncu --metrics dram__bytes_read.sum,lts__t_sector_hit_rate.pct,gpu__time_duration.sum --clock-control none -k regex:bench --csv --log-file gpurun_out/s5a_fetch_$g.csv tools/microbench_fetch $g > /dev/null 2>&1
python - <<P
import csv
rows=list(csv.reader(open('gpurun_out/s5a_fetch_$g.csv')))
i=[k for k,r in enumerate(rows) if 'Kernel Name' in r][0]
h=rows[i]
for r in rows[i+1:]:
    d=dict(zip(h,r))
    print($g, d['Kernel Name'][:12], d['Metric Name'], d['Metric Value'], d['Metric Unit'])
P
done
