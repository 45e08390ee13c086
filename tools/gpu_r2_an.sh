# STAGED pack/unpack kernels: bandwidth from ncu (single process, 2 GPUs)
mkdir -p gpurun_out/an
timeout 300 python tools/staged_pack.py 6 > gpurun_out/an/run.txt 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:copy_runs -c 12 --csv python tools/staged_pack.py 2 > gpurun_out/an/ncu.csv 2>gpurun_out/an/ncu.err
cat gpurun_out/an/run.txt
python - <<'PY'
import csv
rows=[r for r in csv.reader(open('gpurun_out/an/ncu.csv')) if len(r)>5]
h=rows[0]; rows=rows[1:]
k={}
for r in rows:
    d=dict(zip(h,r)); key=(d['ID'],d['Device'] if 'Device' in d else '')
    k.setdefault(key,{})[d['Metric Name']]=(float(d['Metric Value'].replace(',','')),d['Metric Unit'])
for key,m in sorted(k.items(), key=lambda x:int(x[0][0])):
    t=m['gpu__time_duration.sum']; rd=m['dram__bytes_read.sum']; wr=m['dram__bytes_write.sum']
    scale={'ns':1e-9,'us':1e-6,'usecond':1e-6,'nsecond':1e-9,'ms':1e-3,'msecond':1e-3}[t[1]]
    bs={'byte':1,'Kbyte':1e3,'Mbyte':1e6,'Gbyte':1e9}
    b=rd[0]*bs[rd[1]]+wr[0]*bs[wr[1]]
    print(key, f"{t[0]*scale*1e6:.1f} us  dram {b/1e6:.1f} MB  {b/(t[0]*scale)/1e9:.0f} GB/s")
PY
