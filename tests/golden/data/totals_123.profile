dreamsched-profile v1
1	all	0	1000000	2000000	3000000
link	1.0	0
