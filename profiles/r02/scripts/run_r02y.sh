for rep in 1 2; do
for lib in default build_variants/libodpo_h00.so build_variants/libodpo_h12.so build_variants/libodpo_h10_g16.so; do
  timeout 600 python profiles/r02/lmhead_fwd_ab.py $lib 2>&1 | tail -1
done
done
timeout 900 ncu --metrics dram__bytes_read.sum,gpu__time_duration.sum,sm__cycles_elapsed.avg.per_second,lts__t_sector_hit_rate.pct --clock-control none -k regex:"k_lmhead_fwd2" -s 2 -c 1 python -c "
import torch, sys; sys.path.insert(0,'.')
import paper_2410_18252_b200 as odpo
B,T,d,V=128,1024,4096,128256
g=torch.Generator(device='cuda').manual_seed(0)
hid=(torch.randint(-32,32,(B,T,d),device='cuda',generator=g).float()/32).to(torch.bfloat16)
Wh=(torch.randint(-32,32,(V,d),device='cuda',generator=g).float()/256).to(torch.bfloat16)
tok=torch.randint(0,V,(B,T),device='cuda',generator=g,dtype=torch.int32); msk=torch.ones((B,T),dtype=torch.uint8,device='cuda')
for _ in range(3): odpo.lmhead_seq_logprobs(hid,Wh,tok,msk)
torch.cuda.synchronize()
" 2>&1 | grep -E "dram__bytes|duration|cycles_elapsed|hit_rate"
