import subprocess, itertools
g7=[-999424, 1097728, 573440, 2146304]; g14=[-458752, 589824, 589824, 589824]; g15=[0,0,524288,0]
e2=[0,0,1,0]
# n: need sphere data; use dummy n (only used for all-radical D4)
line=' '.join(map(str,[1]+g7+[0,0,0,7]))+' '+' '.join(map(str,[0]+e2+[0,0,0,18]))+' '+' '.join(map(str,[1]+g14+[0,0,0,14]))+' '+' '.join(map(str,[1]+g15+[0,0,0,15]))
print(subprocess.run([__import__('sys').argv[1]],input=line+'\n',capture_output=True,text=True).stdout)
