# Build libgnb.so (sm_100a) and the CPU oracle.  `python -c "import __graft_entry__ as g; g.build()"` runs the same.
NVCC ?= nvcc
ARCH := -gencode arch=compute_100a,code=sm_100a
NVFLAGS := $(ARCH) -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Xcompiler -O3
PKG := paper_1905_13746_b200
CU := predict predict_i32_exact predict_i32_fma predict_u16_exact predict_u16_fma \
      predict_u8_exact predict_u8_fma fit gen gather sort fin_select api
CXX_SRC := fin ingest comms narrow
OBJDIR := $(PKG)/csrc/build
OBJ := $(CU:%=$(OBJDIR)/%.o) $(CXX_SRC:%=$(OBJDIR)/%.o)
HDR := $(wildcard $(PKG)/csrc/*.h $(PKG)/csrc/*.cuh) include/gnb.h

PYINC := $(shell python3 -c "import sysconfig; print(sysconfig.get_paths()['include'])")
PYEXT := $(shell python3 -c "import sysconfig; print(sysconfig.get_config_var('EXT_SUFFIX'))")
ADAPT := $(PKG)/_adapt$(PYEXT)

all: $(PKG)/libgnb.so $(ADAPT) oracle

$(ADAPT): $(PKG)/csrc/adapt.cpp
	g++ -O3 -std=c++17 -ffp-contract=off -fPIC -shared -I$(PYINC) -o $@ $<

# one object per translation unit so `make -j` compiles the K-PRED instances in parallel
$(OBJDIR)/%.o: $(PKG)/csrc/%.cu $(HDR)
	@mkdir -p $(OBJDIR)
	$(NVCC) $(NVFLAGS) -c -o $@ $<

$(OBJDIR)/%.o: $(PKG)/csrc/%.cpp $(HDR)
	@mkdir -p $(OBJDIR)
	$(NVCC) $(NVFLAGS) -c -o $@ $<

$(PKG)/libgnb.so: $(OBJ)
	$(NVCC) $(NVFLAGS) -shared -o $@ $(OBJ) -ldl

oracle:
	$(MAKE) -C oracle

clean:
	rm -f $(PKG)/libgnb.so $(ADAPT)
	rm -rf $(OBJDIR)
	$(MAKE) -C oracle clean

.PHONY: all oracle clean
