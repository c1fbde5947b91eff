# Build libgnb.so (sm_100a) and the CPU oracle.  `python -c "import __graft_entry__ as g; g.build()"` runs the same.
NVCC ?= nvcc
ARCH := -gencode arch=compute_100a,code=sm_100a
NVFLAGS := $(ARCH) -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Xcompiler -O3
PKG := paper_1905_13746_b200
SRC := $(PKG)/csrc/predict.cu $(PKG)/csrc/fit.cu $(PKG)/csrc/gen.cu $(PKG)/csrc/gather.cu $(PKG)/csrc/sort.cu $(PKG)/csrc/fin_select.cu $(PKG)/csrc/api.cu $(PKG)/csrc/fin.cpp $(PKG)/csrc/ingest.cpp
HDR := $(wildcard $(PKG)/csrc/*.h $(PKG)/csrc/*.cuh) include/gnb.h

PYINC := $(shell python3 -c "import sysconfig; print(sysconfig.get_paths()['include'])")
PYEXT := $(shell python3 -c "import sysconfig; print(sysconfig.get_config_var('EXT_SUFFIX'))")
ADAPT := $(PKG)/_adapt$(PYEXT)

all: $(PKG)/libgnb.so $(ADAPT) oracle

$(ADAPT): $(PKG)/csrc/adapt.cpp
	g++ -O3 -std=c++17 -fPIC -shared -I$(PYINC) -o $@ $<

$(PKG)/libgnb.so: $(SRC) $(HDR)
	$(NVCC) $(NVFLAGS) -shared -o $@ $(SRC)

oracle:
	$(MAKE) -C oracle

clean:
	rm -f $(PKG)/libgnb.so $(ADAPT)
	$(MAKE) -C oracle clean

.PHONY: all oracle clean
