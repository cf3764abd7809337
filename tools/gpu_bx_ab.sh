# boxcar prefix variants (build/ab/<v> copies + the working tree): kernel launch times (ncu
# launch list of 3 config-B chunk-0 runs) and config-B file search wall times
set -x
for v in build/ab/old build/ab/mask . ; do
  tag=$(basename $v)
  (cd $v && timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:boxcar_prefix -c 6 --csv --log-file $GRAFT_REPO_ROOT/gpurun_out/bxab_$tag.csv python tools/profile_chunk.py 6 > /dev/null 2>&1)
  grep -o '"[0-9]*"$' gpurun_out/bxab_$tag.csv | tr '\n' ' '; echo " <- $tag"
done
for r in 1 2; do for v in build/ab/mask . ; do
  (cd $v && timeout 600 python -c "
import sys,time,torch; sys.path.insert(0,'.')
import bench
from paper_2512_00398_b200.engine import Engine
cfg=dict(bench.CONFIG_B); task=bench.build_task(cfg); pl=bench.make_payload(cfg, task.plan)
with Engine(0) as e:
    for _ in range(2): e.search_file(pl, cfg['nsamples'], task.chunks, task.plan, task.engine)
    torch.cuda.synchronize(); t=[]
    for _ in range(8):
        t0=time.perf_counter(); e.search_file(pl, cfg['nsamples'], task.chunks, task.plan, task.engine); torch.cuda.synchronize(); t.append(time.perf_counter()-t0)
print('$v', sorted(t)[4]*1e3)
")
done; done
