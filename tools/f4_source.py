import sys, subprocess, os
import paper_2106_04284_b200 as llama, workloads as W
EXT=[4096,4096]
cases=[("aos","row","aos","col"),("aos","row","soa_mb","col"),("soa_mb","col","soa_mb","row"),("aos","row","aos","morton"),("soa_mb","morton","aos","col"),("soa_mb","row","aos","col")]
for sk,sl,dk,dl in cases:
    sm=llama.Mapping.from_spec(W.PARTICLE7,EXT,(sk,1,False),lin=sl)
    dm=llama.Mapping.from_spec(W.PARTICLE7,EXT,(dk,1,False),lin=dl)
    pl=llama.plan(sm,dm)
    src=llama.plan_source(sm,dm)
    defs=[l for l in src.splitlines() if l.startswith("#define LLB_") and any(x in l for x in ("BMAP","LLB_P ","TY ","BLOCK","NS ","ND ","MINB"))]
    fn=f"/tmp/f4_{sk}{sl}_{dk}{dl}.cu"; open(fn,"w").write(src)
    r=subprocess.run(["/usr/local/cuda/bin/nvcc","-gencode","arch=compute_100a,code=sm_100a","-cubin","-std=c++17","-Xptxas","-v","-o",fn+".cubin",fn],capture_output=True,text=True)
    regs=[l for l in r.stderr.splitlines() if "registers" in l or "spill" in l]
    print(sk,sl,dk,dl,pl['jit'],defs, r.returncode, regs[-2:] if regs else r.stderr[-500:])
