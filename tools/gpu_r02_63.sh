export PATH=/usr/local/cuda/bin:$PATH
timeout 900 python tools/cosched.py --config c2 --steps 200 --tunes "nf=1;nf=0;nf=1;nf=0;sol=2;sol=4" 2>&1 | grep levels | cut -c1-400
